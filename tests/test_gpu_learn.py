"""GPU parity of the distortion-gradient kernel (iq_distortion_grad, R29)
against the fp64 oracle, element by element, and a short learning loop
through the C ABI (GPU gradient -> host chain rule -> explicit parameters).

Per-element tolerance on dL/dM_b[i][j] = 2 sum_rows e_i xbar_j, derived from
the arithmetic: (1) the kernel's fp32 row math (normalisation, rotation,
e = ybar - C[code]) carries ~1e-6 relative error on each product, so
5e-5 * 2 sum_rows |e_i| |xbar_j| bounds the accumulated rounding; (2) a
decision taken on the other side of a threshold (the parity bar allows it
within 1e-5 of a threshold) moves that row's e_i by the centroid gap dC, so
every oracle coordinate within 1e-5 of a threshold adds 2 dC |xbar_j| to its
elements' allowance.  The distortion agrees to 1e-4 relative."""
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
    Go = Lo.operator_grad(X, po)
    Gg = grad.cpu().numpy().reshape(Go.shape)
    xb, yb, e = Lo._blocks(X, po)
    scale = 2.0 * np.einsum("ngi,ngj->gij", np.abs(e), np.abs(xb))
    T = po.cb.thresholds
    near = np.min(np.abs(yb[..., None] - T), axis=-1) <= 1e-5              # [n, g, w]
    gap = float(np.max(np.diff(po.cb.centroids)))
    flip = 2.0 * gap * np.einsum("ngi,ngj->gij", near.astype(np.float64), np.abs(xb))
    err = np.abs(Gg - Go)
    tol = 5e-5 * scale + flip + 1e-12
    assert np.all(err <= tol), float(np.max(err / tol))
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
