"""Out-of-bounds write checks with canaries (compute-sanitizer is not available
on the GPU pool): every output of the code-emitting kernels is a view into a
larger buffer filled with a canary pattern; after the launch the bytes before
and after the view must be untouched, and the view itself must hold what the
kernel owes (checked against an unguarded launch, which the parity tests
compare with the oracle).  Ragged row counts exercise the tail tiles and the
byte-piece code stores ("Code stores"); the append kernel
is checked at the first and last cache positions of every slot.
"""
import numpy as np
import pytest
import torch

import iqsynth
import paper_2603_28430_b200 as iq

pytestmark = pytest.mark.gpu

PAD = 64          # canary rows on each side
CAN8 = 0xA5       # canary byte
CANF = -12345.5   # canary float


def _guarded(shape, dtype, fill):
    big = torch.full((shape[0] + 2 * PAD,) + tuple(shape[1:]), fill, dtype=dtype, device="cuda")
    return big, big[PAD:PAD + shape[0]]


def _intact(big, n, fill):
    head, tail = big[:PAD], big[PAD + n:]
    return bool(torch.all(head == fill)) and bool(torch.all(tail == fill))


@pytest.mark.parametrize("dt", [iq.F16, iq.F32])
@pytest.mark.parametrize("d", [64, 128, 512])
@pytest.mark.parametrize("bits", [1, 2, 3, 4])
@pytest.mark.parametrize("n", [1, 33, 4097])
def test_encoder_outputs_stay_in_bounds(dt, d, bits, n):
    p = iq.iq_make_params(d, bits, iq.FULL, iqsynth.PARAMS_SEED, device=0)
    tdt = torch.float16 if dt == iq.F16 else torch.float32
    x = torch.from_numpy(iqsynth.unit_vectors(n, d, 500 + n, np.float32)).to("cuda", tdt)
    ref_c, ref_n = iq.iq_quantize(p, x)
    ref_y = iq.iq_roundtrip(p, x)
    # quantize
    cb, c = _guarded((n, p.code_bytes), torch.uint8, CAN8)
    nb, nm = _guarded((n,), torch.float32, CANF)
    iq.iq_quantize(p, x, c, nm)
    torch.cuda.synchronize()
    assert _intact(cb, n, CAN8) and _intact(nb, n, CANF)
    assert torch.equal(c, ref_c) and torch.equal(nm, ref_n)
    # fused roundtrip, values only (the bench's kernel) and with codes
    yb, y = _guarded((n, d), tdt, CANF)
    iq.iq_roundtrip(p, x, y=y)
    torch.cuda.synchronize()
    assert _intact(yb, n, CANF) and torch.equal(y, ref_y)
    cb2, c2 = _guarded((n, p.code_bytes), torch.uint8, CAN8)
    nb2, nm2 = _guarded((n,), torch.float32, CANF)
    yb2, y2 = _guarded((n, d), tdt, CANF)
    iq.iq_roundtrip(p, x, y=y2, codes=c2, norms=nm2)
    torch.cuda.synchronize()
    assert _intact(cb2, n, CAN8) and _intact(nb2, n, CANF) and _intact(yb2, n, CANF)
    assert torch.equal(c2, ref_c) and torch.equal(nm2, ref_n)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("n", [1, 129, 1000])
def test_stage2_outputs_stay_in_bounds(d, bits, n):
    p = iq.iq_make_params_qjl(d, bits, iq.FULL, iqsynth.PARAMS_SEED, device=0)
    x = torch.from_numpy(iqsynth.unit_vectors(n, d, 900 + n, np.float32)).to("cuda", torch.float16)
    rc, rn, rq, rg = iq.iq_quantize_qjl(p, x)
    cb, c = _guarded((n, p.code_bytes), torch.uint8, CAN8)
    nb, nm = _guarded((n,), torch.float32, CANF)
    qb, qj = _guarded((n, d // 8), torch.uint8, CAN8)
    gb, gm = _guarded((n,), torch.float32, CANF)
    iq.iq_quantize_qjl(p, x, c, nm, qj, gm)
    torch.cuda.synchronize()
    assert _intact(cb, n, CAN8) and _intact(nb, n, CANF) and _intact(qb, n, CAN8) and _intact(gb, n, CANF)
    assert torch.equal(c, rc) and torch.equal(nm, rn) and torch.equal(qj, rq) and torch.equal(gm, rg)


@pytest.mark.parametrize("dt", [iq.F16, iq.F32])
@pytest.mark.parametrize("d", [64, 128, 256])
@pytest.mark.parametrize("bits", [1, 3, 4])
def test_append_writes_only_its_slot_position(dt, d, bits):
    slots, cap = 37, 5
    p = iq.iq_make_params(d, bits, iq.FULL, iqsynth.PARAMS_SEED, device=0)
    tdt = torch.float16 if dt == iq.F16 else torch.float32
    x = torch.from_numpy(iqsynth.unit_vectors(slots, d, 77, np.float32)).to("cuda", tdt)
    ref_c, ref_n = iq.iq_quantize(p, x)
    for pos in (0, cap - 1):
        codes = torch.full((slots, cap, p.code_bytes), CAN8, dtype=torch.uint8, device="cuda")
        norms = torch.full((slots, cap), CANF, dtype=torch.float32, device="cuda")
        iq.iq_append_kv(p, x, codes, norms, position=pos)
        torch.cuda.synchronize()
        other = [q for q in range(cap) if q != pos]
        assert bool(torch.all(codes[:, other] == CAN8)) and bool(torch.all(norms[:, other] == CANF))
        assert torch.equal(codes[:, pos], ref_c) and torch.equal(norms[:, pos], ref_n)
