"""C-ABI contract tests that need no GPU: the library loads, exports every
symbol include/isoquant.h declares, validates arguments, and its host-side
parameter builder agrees with the oracle's independent re-derivation."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def iq():
    from __graft_entry__ import load_builder
    _build = load_builder()
    _build.build()
    import paper_2603_28430_b200 as m
    return m


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "isoquant.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(iq_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(iq):
    names = _declared_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(iq.lib, name), name


def test_version_and_status_strings(iq):
    assert "sm_100a" in iq.iq_version()
    assert iq.lib.iq_abi_version() == 1
    for s, name in [(0, b"IQ_OK"), (2, b"IQ_ERR_UNSUPPORTED"), (4, b"IQ_ERR_DEVICE_MISMATCH")]:
        assert iq.lib.iq_status_string(s) == name


def test_code_bytes(iq):
    assert iq.iq_code_bytes_per_vector(128, 3) == 48
    assert iq.iq_code_bytes_per_vector(512, 4) == 256
    assert iq.iq_code_bytes_per_vector(7, 3) == 3


def test_invalid_arguments(iq):
    h = ctypes.c_void_p()
    for d, b, v in [(0, 3, 0), (128, 0, 0), (128, 5, 0), (128, 3, 3)]:
        assert iq.lib.iq_make_params(d, b, v, 1, -1, ctypes.byref(h)) == 1
        assert iq.lib.iq_last_error_detail()
    assert iq.lib.iq_make_params(128, 3, 0, 1, -1, None) == 1
    assert iq.lib.iq_free_params(None) == 0


def test_host_only_handle_rejects_compute(iq):
    p = iq.iq_make_params(128, 3, iq.FULL, 1, device=-1)
    buf = ctypes.c_void_p(16)
    st = iq.lib.iq_roundtrip(p.handle, 1, 4, buf, buf, None, None, None)
    assert st == 4  # IQ_ERR_DEVICE_MISMATCH, before any CUDA call
    assert iq.lib.iq_roundtrip(None, 1, 4, buf, buf, None, None, None) == 1
    assert iq.lib.iq_quantize(p.handle, 7, 4, buf, buf, buf, None) == 1   # bad dtype


def test_gpu_handle_fails_loudly_without_gpu(iq):
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    h = ctypes.c_void_p()
    st = iq.lib.iq_make_params(128, 3, 0, 1, 0, ctypes.byref(h))
    assert st in (5, 6) and not h.value
    assert iq.lib.iq_last_error_detail()
    with pytest.raises(iq.IQError):
        iq.iq_make_params(128, 3, iq.FULL, 1, device=0)


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("d", [32, 128, 512, 7])
def test_params_match_oracle_rederivation(iq, variant, d):
    """The library's host generator and the oracle's independent Python
    re-derivation of reading [R12] give the same canonical parameters."""
    from oracle import iq_oracle as O
    seed = 20260331
    p = iq.iq_make_params(d, 3, variant, seed, device=-1)
    ex = iq.iq_export_params(p)
    qL, qR, cs = O.make_rotation_params(d, variant, seed)
    if variant == O.FULL:
        ref = np.concatenate([qL, qR], axis=1).reshape(-1)
    elif variant == O.FAST:
        ref = qL.reshape(-1)
    else:
        ref = cs.reshape(-1)
    assert ex["rot"].shape == ref.shape
    assert np.max(np.abs(ex["rot"] - ref)) <= 1e-15


@pytest.mark.parametrize("bits", [1, 2, 3, 4])
@pytest.mark.parametrize("d", [32, 128, 256, 512])
def test_codebook_matches_oracle(iq, bits, d):
    from oracle import iq_oracle as O
    p = iq.iq_make_params(d, bits, 0, 1, device=-1)
    ex = iq.iq_export_params(p)
    cb = O.make_codebook(d, bits)
    assert np.array_equal(ex["centroids"].astype(np.float64), cb.centroids)
    # the library stores fp32 thresholds: the oracle's exact midpoints rounded once [R14b]
    assert np.array_equal(ex["thresholds"], cb.thresholds.astype(np.float32))


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_block_operator_is_the_sandwich_map(iq, variant):
    """The fp32 operator the kernels apply equals the oracle's block map on
    the basis vectors, to fp32 rounding."""
    from oracle import iq_oracle as O
    d = 64
    p = iq.iq_make_params(d, 2, variant, 77, device=-1)
    m = iq.iq_export_block_matrices(p)
    po = O.make_params(d, 2, variant, 77)
    w = O.block_width(variant)
    g = d // w
    M = m.reshape(g, w, w).astype(np.float64)
    for b in range(g):
        for j in range(w):
            e = np.zeros((1, 1, w)); e[0, 0, j] = 1.0
            if variant == O.PLANAR2D:
                col = O.forward_blocks(variant, None, None, po.cs[b:b + 1], e)
            else:
                col = O.forward_blocks(variant, po.qL[b:b + 1], None if po.qR is None else po.qR[b:b + 1], None, e)
            assert np.allclose(M[b][:, j], col.reshape(-1), atol=6e-8, rtol=0)


def test_qjl_sketch_generator_matches_oracle(iq):
    """The C++ stage-2 sketch generator (params.cpp, R20) and the oracle's
    independent re-derivation give the same fp16 matrix."""
    from oracle import qjl_oracle as Q
    for d in (16, 64):
        p = iq.iq_make_params_qjl(d, 3, iq.FULL, 20260331, device=-1)
        assert np.array_equal(iq.iq_export_qjl_matrix(p).astype(np.float64), Q.sketch_matrix(d, 20260331))
    assert iq.iq_qjl_bytes_per_vector(128) == 16
    p = iq.iq_make_params(64, 3, iq.FULL, 1, device=-1)
    with pytest.raises(iq.IQError):
        iq.iq_export_qjl_matrix(p)


def test_param_sets_generator_matches_oracle(iq):
    """Set s of a multi-set handle is exactly the seed + s parameters (R31)."""
    from oracle import iq_oracle as O
    p = iq.iq_make_params_sets(64, 3, iq.FULL, 20260331, 3, 256, device=-1)
    for s in range(3):
        want = iq.iq_export_params(iq.iq_make_params(64, 3, iq.FULL, 20260331 + s, device=-1))["rot"]
        assert np.array_equal(iq.iq_export_params_set(p, s), want)
        qL, qR, _ = O.make_rotation_params(64, O.FULL, 20260331 + s)
        assert np.allclose(want.reshape(-1, 8)[:, :4], qL, atol=1e-15)
    # any set_rows >= 1 (finer sets serve iq_append_kv / the consumer; the
    # batch kernels refuse them at call time, tests/test_gpu_append.py)
    iq.iq_make_params_sets(64, 3, iq.FULL, 1, 2, 100, device=-1)
    with pytest.raises(iq.IQError):
        iq.iq_make_params_sets(64, 3, iq.FULL, 1, 2, 0, device=-1)       # set_rows < 1
    with pytest.raises(iq.IQError):
        iq.iq_export_params_set(p, 3)
