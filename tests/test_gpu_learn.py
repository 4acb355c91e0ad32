"""GPU parity of the distortion-gradient kernel (iq_distortion_grad, R29)
against the fp64 oracle, and a short learning loop through the C ABI
(GPU gradient -> host chain rule -> explicit parameters).  Tolerance:
Frobenius-relative 1e-3 on dL/dM (fp32 per-row math; a decision taken on the
other side of a threshold -- allowed for 1e-4 of coordinates -- moves that
row's contribution by 2 dC xbar, which is large against the small b = 4
gradient) and 1e-4 on the distortion."""
import numpy as np
import pytest

import iqsynth
from oracle import iq_oracle as O
from oracle import learn_oracle as Lo

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2603_28430_b200 as iq  # noqa: E402

SEED = iqsynth.PARAMS_SEED
NP = {iq.F32: np.float32, iq.F16: np.float16}


@pytest.mark.parametrize("dt", [iq.F32, iq.F16])
@pytest.mark.parametrize("variant", [iq.FULL, iq.FAST, iq.PLANAR2D])
@pytest.mark.parametrize("d", [64, 128, 256, 512])
@pytest.mark.parametrize("bits", [2, 3, 4])
def test_grad_parity(bits, d, variant, dt):
    n = 4096 + 33
    X = iqsynth.outlier_vectors(n, d, 50 + bits + d, np.float64).astype(NP[dt])
    p = iq.iq_make_params(d, bits, variant, SEED, device=0)
    grad, loss = iq.iq_distortion_grad(p, torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    po = O.make_params(d, bits, variant, SEED)
    Go = Lo.operator_grad(X, po).reshape(-1)
    Gg = grad.cpu().numpy()
    assert np.linalg.norm(Gg - Go) <= 1e-3 * np.linalg.norm(Go), np.linalg.norm(Gg - Go) / np.linalg.norm(Go)
    Lw = Lo.distortion(X, po)
    assert abs(float(loss) - Lw) <= 1e-4 * Lw


def test_learning_loop_lowers_distortion():
    """Ten projected-gradient steps on outlier-channel rows (the unequal-energy
    case the rotation is for) lower the distortion."""
    d, bits = 128, 2
    X = torch.from_numpy(iqsynth.outlier_vectors(1 << 16, d, 77, np.float32)).cuda()
    p = iq.iq_make_params(d, bits, iq.FULL, SEED, device=0)
    rot = iq.iq_export_params(p)["rot"]
    losses = []
    for _ in range(10):
        grad, loss = iq.iq_distortion_grad(p, X)
        losses.append(float(loss))
        g = iq.iq_rot_grad_from_operator_grad(p, grad.cpu().numpy())
        rot = rot - 0.05 * g / np.linalg.norm(g) * np.sqrt(rot.size / 8)
        p = iq.iq_make_params_explicit(d, bits, iq.FULL, rot, device=0)
    _, loss = iq.iq_distortion_grad(p, X)
    losses.append(float(loss))
    assert losses[-1] < losses[0], losses
    # the learned handle quantizes like any other (roundtrip MSE follows the distortion)
    y = iq.iq_roundtrip(p, X)
    assert torch.isfinite(y).all()
