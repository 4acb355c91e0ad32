"""The GPU parity harness (tests/iq_parity.py) pinned on CPU: it must accept
the oracle's own outputs (cast to the kernel's storage dtype) and reject the
failures a kernel could plausibly produce -- one wrong code far from a
threshold, one garbage row, one row scaled by 1 %, one nonzero output for a
zero row -- with no row exempt.  Test infrastructure only."""
import numpy as np
import pytest

import iqsynth
import iq_parity as parity
from oracle import iq_oracle as O


def _case(variant, dt, d=128, bits=3, n=512):
    X = iqsynth.unit_vectors(n, d, 5, dt)
    X[0] = 0.0                                       # a zero row (x^ = 0 exactly)
    po = O.make_params(d, bits, variant, 1)
    xh, codes, packed, rho = O.roundtrip(X, po)
    return X, po, xh, codes, rho


@pytest.mark.parametrize("dt", [np.float16, np.float32])
@pytest.mark.parametrize("variant", [O.FULL, O.FAST, O.PLANAR2D])
@pytest.mark.parametrize("bits", [2, 4])
def test_values_accept_oracle_output(variant, dt, bits):
    X, po, xh, _, _ = _case(variant, dt, bits=bits)
    parity.assert_values(parity.check_values(X, po, xh.astype(dt), dt), dt)


def _far_coordinate(X, po):
    """(row, coordinate) farthest from every threshold (a code error there is
    not a boundary effect)."""
    y = O.rotated_coordinates(X, po)
    dist = np.min(np.abs(y[..., None] - po.cb.thresholds), axis=-1)
    dist[0] = 0.0
    i, j = np.unravel_index(np.argmax(dist), dist.shape)
    return int(i), int(j)


@pytest.mark.parametrize("dt", [np.float16, np.float32])
def test_values_reject_one_wrong_code(dt):
    X, po, xh, codes, rho = _case(O.FULL, dt)
    i, j = _far_coordinate(X, po)
    bad = codes.copy()
    bad[i, j] = bad[i, j] + 1 if bad[i, j] + 1 < po.L else bad[i, j] - 1
    y = O.decode(bad, rho, po).astype(dt)
    with pytest.raises(AssertionError):
        parity.assert_values(parity.check_values(X, po, y, dt), dt)


@pytest.mark.parametrize("dt", [np.float16, np.float32])
def test_values_reject_garbage_row_and_scaled_row(dt):
    X, po, xh, _, _ = _case(O.FAST, dt)
    y = xh.astype(dt)
    y[7] = iqsynth.unit_vectors(1, X.shape[1], 99, dt)[0]
    with pytest.raises(AssertionError):
        parity.assert_values(parity.check_values(X, po, y, dt), dt)
    y = xh.copy()
    y[9] *= 1.01
    with pytest.raises(AssertionError):
        parity.assert_values(parity.check_values(X, po, y.astype(dt), dt), dt)


def test_values_reject_nonzero_zero_row():
    X, po, xh, _, _ = _case(O.FULL, np.float16)
    y = xh.astype(np.float16)
    y[0, 5] = np.float16(1e-4)
    with pytest.raises(AssertionError):
        parity.assert_values(parity.check_values(X, po, y, np.float16), np.float16)


def test_decode_check():
    X, po, xh, codes, rho = _case(O.PLANAR2D, np.float32, d=64)
    packed = O.pack_codes(codes, po.bits)
    assert parity.check_decode(packed, rho.astype(np.float32), xh.astype(np.float32), po) <= 1e-6
    y = xh.copy()
    y[3, :4] = -y[3, :4]
    assert parity.check_decode(packed, rho.astype(np.float32), y, po) > 1e-2
