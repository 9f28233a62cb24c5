"""CPU-side checks of the C ABI: the library loads, exports every symbol include/librfr.h declares,
plans workspaces and rejects bad arguments before touching a device (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "librfr.h")


def _lib():
    from paper_2605_29097_b200 import rfr
    if not os.path.exists(rfr.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build_librfr()
    return rfr, rfr.load()


def declared_symbols():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rfr_[a-z_]+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("rfr_forward", "rfr_filter", "rfr_backward", "rfr_workspace_size"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    rfr, lib = _lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(rfr.EXPORTS)
    assert lib.rfr_abi_version() == 2
    assert lib.rfr_status_string(2) == b"shape mismatch or workspace too small"


def test_workspace_plan_is_sane():
    rfr, lib = _lib()
    n = rfr.rfr_workspace_size(1 << 20, 16384, 256, 1 << 20)
    # records (48 B/sample) + backward partial sums + split buffers, capped at a few GiB
    assert 48 * (1 << 20) < n < 8 << 30
    assert rfr.rfr_workspace_size(0, 0, 1, 0) >= 256
    small = rfr.rfr_workspace_size(4096, 64, 64, 4096)
    assert small < n
    out = C.c_size_t()
    assert lib.rfr_workspace_size(-1, 1, 1, 0, C.byref(out)) == 2
    assert lib.rfr_workspace_size(1, 1, 9000, 0, C.byref(out)) == 2   # n_freq > 8192 unsupported


def test_argument_errors_before_any_launch():
    rfr, lib = _lib()
    g = rfr.rfr_freq_grid(77e9, 1e6, 8)
    # null sample struct / null workspace -> RFR_E_ARG without touching a device
    assert lib.rfr_forward(None, 1.0, None, C.byref(g), None, None, None, None) == 1
    s = rfr.rfr_samples()
    s.n_rays, s.n_per_ray = 1, 1
    a = rfr.rfr_antennas()
    assert lib.rfr_forward(C.byref(s), 1.0, C.byref(a), C.byref(g), None, None, None, None) == 1
    w = rfr.rfr_workspace(None, 0, 1, 1, 8, 0)
    assert lib.rfr_loss(None, None, 0, None, None, C.byref(w), None) == 1
    assert lib.rfr_filter_power(None, 4, None, None) == 1
    assert lib.rfr_filter_power(None, 0, None, None) == 0


def test_no_cpu_fallback():
    import torch
    rfr, _ = _lib()
    t = torch.zeros(4)
    with pytest.raises(rfr.RfrError):
        rfr._ptr(t)


def test_shard_range_partitions():
    rfr, _ = _lib()
    for n in (0, 1, 7, 64, 16384, 16385):
        for w in (1, 2, 3, 4, 8):
            rs = [rfr.shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1


def test_workspace_planned_dims_bound_every_call():
    """a call with more antennas or more bins than the workspace was planned for is a
    shape error (RFR_E_SHAPE) before any launch -- the per-antenna and per-bin regions are sized
    from the planning dimensions.  Host pointers stand in for device ones: nothing is launched."""
    rfr, lib = _lib()
    import numpy as np
    na, nf, ns = 4, 8, 4
    plan = dict(n_samples=ns, n_ant=na, n_freq=nf, n_query=ns)
    nbytes = rfr.rfr_workspace_size(ns, na, nf, ns)
    fake = C.c_void_p(0x1000)                           # never dereferenced on these paths
    w = rfr.rfr_workspace(fake, nbytes, plan["n_samples"], plan["n_ant"], plan["n_freq"],
                          plan["n_query"])
    buf = np.zeros(64, np.float32)
    p = C.c_void_p(buf.ctypes.data)
    s = rfr.rfr_samples()
    for f in ("x", "y", "z", "sdf", "refl", "nx", "ny", "nz", "power"):
        setattr(s, f, p)
    s.n_rays, s.n_per_ray = 1, ns

    def ants(n):
        a = rfr.rfr_antennas()
        a.tx_x = a.tx_y = a.tx_z = p
        a.n_ant = n
        return a

    sig = buf.ctypes.data_as(C.c_void_p)
    for n_ant, n_freq in ((na + 1, nf), (na, nf + 1)):
        a, g = ants(n_ant), rfr.rfr_freq_grid(77e9, 1e6, n_freq)
        assert lib.rfr_forward(C.byref(s), 1.0, C.byref(a), C.byref(g), None, sig, C.byref(w),
                               None) == 2
        assert lib.rfr_filter(sig, C.byref(a), C.byref(g), p, p, p, ns, p, None, None, C.byref(w),
                              None) == 2
        assert lib.rfr_filter_backward(p, sig, p, C.c_float(0.0), C.byref(a), C.byref(g), p, p, p,
                                       ns, sig, C.byref(w), None) == 2


def test_tensor_core_kernels_issue_tcgen05_mma():
    """The r2 engine's dense contractions (k2_gexp_tc, k2_bins_tc; rfr_tc_gemm.cu) are compiled to
    5th-generation tensor-core MMAs (UTCHMMA, kind::f16 with A in tensor memory) for sm_100a."""
    import shutil
    import subprocess
    rfr, _ = _lib()
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", rfr.LIB_PATH], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)
    for k in ("k2_gexp_tc", "k2_bins_tc"):
        body = [f for f in funcs if k in f.split("\n")[0]]
        assert body, k
        assert "UTCHMMA" in body[0] and "UTCBAR" in body[0], k
