"""The C ABI library loads, exports every symbol include/retina.h declares, and rejects
host-checkable argument errors synchronously (no GPU needed: nothing is launched)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1709_08610_b200 import build as B
from paper_1709_08610_b200 import retina as rt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "retina.h")


@pytest.fixture(scope="module")
def L():
    B.build()
    return rt.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(retina_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert set(names) == set(rt.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)", out))
    for n in names:
        assert n in exported, n
        assert hasattr(L, n)


def test_status_strings_and_version(L):
    assert L.retina_status_string(0).decode() == "RETINA_OK"
    for s in (1, 2, 3):
        assert L.retina_status_string(s).decode().startswith("RETINA_E")
    assert "sm_100a" in L.retina_version().decode()


def _ev(n=1, offsets=1, hits=16):
    return rt.retina_events(n, offsets, hits, 0.0, 0)


def _f(*v):
    return ctypes.cast((ctypes.c_float * len(v))(*v), ctypes.c_void_p)


def _i(*v):
    return ctypes.cast((ctypes.c_int32 * len(v))(*v), ctypes.c_void_p)


def test_grid_response_validation(L):
    alen = _i(4, 4)
    nodes = ctypes.cast((ctypes.c_void_p * 2)(16, 16), ctypes.c_void_p)
    g = L.retina_grid_response
    assert g(None, 1, 0.5, alen, nodes, 16, None) == rt.RETINA_EINVAL
    ev = _ev()
    assert g(ctypes.byref(ev), 1, 0.0, alen, nodes, 16, None) == rt.RETINA_EINVAL
    assert b"sigma" in L.retina_last_error()
    assert g(ctypes.byref(ev), 1, float("nan"), alen, nodes, 16, None) == rt.RETINA_EINVAL
    assert g(ctypes.byref(ev), 7, 0.5, alen, nodes, 16, None) == rt.RETINA_EINVAL
    assert g(ctypes.byref(ev), 1, 0.5, _i(1, 4), nodes, 16, None) == rt.RETINA_EINVAL
    assert g(ctypes.byref(ev), 1, 0.5, alen, nodes, None, None) == rt.RETINA_EINVAL
    bad = _ev(hits=8)  # misaligned hits
    assert g(ctypes.byref(bad), 1, 0.5, alen, nodes, 16, None) == rt.RETINA_EINVAL
    neg = _ev(n=-1)
    assert g(ctypes.byref(neg), 1, 0.5, alen, nodes, 16, None) == rt.RETINA_EINVAL
    big = _i(65536, 65536)
    assert g(ctypes.byref(ev), 1, 0.5, big, nodes, 16, None) == rt.RETINA_EUNSUPPORTED
    gx = L.retina_grid_response_ex
    assert gx(ctypes.byref(ev), 1, 0.5, alen, nodes, 16, 8, None) == rt.RETINA_EINVAL  # unknown algorithm
    assert gx(ctypes.byref(ev), 1, 0.5, alen, nodes, 16, -1, None) == rt.RETINA_EINVAL
    for algo in (rt.GRID_TENSOR, rt.GRID_TENSOR_F16, rt.GRID_TENSOR_F16_PAIR, rt.GRID_TENSOR_F16_SINGLE,
                 rt.GRID_SEPARABLE):  # LINE2D does not factorise
        assert gx(ctypes.byref(ev), 0, 0.5, alen, nodes, 16, algo, None) == rt.RETINA_EUNSUPPORTED
    e0 = _ev(n=0)  # nothing to launch: every algorithm accepts an empty batch
    for algo in (rt.GRID_AUTO, rt.GRID_DIRECT, rt.GRID_SEPARABLE, rt.GRID_TENSOR, rt.GRID_TENSOR_F16,
                 rt.GRID_TENSOR_F16_PAIR, rt.GRID_TENSOR_F16_SINGLE):
        assert gx(ctypes.byref(e0), 1, 0.5, alen, nodes, 16, algo, None) == rt.RETINA_OK


def test_peaks_validation(L):
    p = L.retina_find_peaks
    assert p(16, 1, 4, _i(4, 4), 0.0, 4, 16, 16, 16, None) == rt.RETINA_EINVAL   # P = 4
    assert p(16, 1, 2, _i(4, 4), 0.0, -1, 16, 16, 16, None) == rt.RETINA_EINVAL  # capacity < 0
    assert p(16, -1, 2, _i(4, 4), 0.0, 4, 16, 16, 16, None) == rt.RETINA_EINVAL
    assert p(16, 1, 2, _i(1, 4), 0.0, 4, 16, 16, 16, None) == rt.RETINA_EINVAL
    assert p(16, 0, 2, _i(4, 4), 0.0, 4, 16, 16, 16, None) == rt.RETINA_OK       # nothing to do
    assert p(16, 1, 2, _i(4, 4), float("nan"), 4, 16, 16, 16, None) == rt.RETINA_EINVAL


def test_peaks_workspace_size_and_validation(L):
    sz = L.retina_find_peaks_workspace_size
    sz.restype = ctypes.c_size_t
    # 1024^2 cells -> 8 slabs of 131072 cells per event; per slab a count (4 B) and a list of
    # 1024 (index, value) pairs (8 B each)
    per_slab = 4 + 1024 * 8
    assert sz(10, 2, _i(1024, 1024)) == 10 * 8 * per_slab
    # P = 3 grids are scanned in memory order (n2, n0, n1) (z0 planes outermost, Z37).
    # Rows (axis_len[1] cells) of a multiple of 4 cells (<= 2048): the plane-block path
    # (peaks3.cu): per segment (z0 plane, block of 2048 / n1 rows) a count, an offset and 32
    # (index, value) pairs (plus one int per chunk of 512 segments for the pass-2 chunk totals)
    per_seg = 2 * 4 + 32 * 8
    assert sz(3, 3, _i(256, 256, 256)) == 3 * (256 * 32) * per_seg + 3 * 16 * 4
    assert sz(2, 3, _i(23, 28, 19)) == 2 * (19 * 1) * per_seg + 2 * 1 * 4  # 73 rows cover the 23: one block
    assert sz(1, 3, _i(20, 30, 29)) == 1 * 1 * per_slab                  # 30 % 4 != 0: slab path
    assert sz(0, 2, _i(4, 4)) == 0 and sz(1, 4, _i(4, 4)) == 0
    p = L.retina_find_peaks_ws
    p.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_float, ctypes.c_int32,
                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    assert p(16, 2, 2, _i(1024, 1024), 0.0, 4, 16, 16, 16, 16, 8, None) == rt.RETINA_EINVAL  # too small
    assert b"workspace" in L.retina_last_error()
    assert p(16, 2, 2, _i(1024, 1024), 0.0, 4, 16, 16, 16, None, 1 << 20, None) == rt.RETINA_EINVAL
    assert p(16, 0, 2, _i(1024, 1024), 0.0, 4, 16, 16, 16, None, 0, None) == rt.RETINA_OK


def test_multistart_validation(L):
    m = L.retina_multistart_optimize
    ev = _ev()
    lo, hi = _f(-1, -1), _f(1, 1)
    assert m(ctypes.byref(ev), 1, 0.5, 8, 16, -1, 0.1, lo, hi, 16, 16, None, None) == rt.RETINA_EINVAL
    assert m(ctypes.byref(ev), 1, 0.5, -8, 16, 1, 0.1, lo, hi, 16, 16, None, None) == rt.RETINA_EINVAL
    assert m(ctypes.byref(ev), 1, 0.5, 8, 16, 1, 0.1, hi, lo, 16, 16, None, None) == rt.RETINA_EINVAL
    assert m(ctypes.byref(ev), 1, 0.5, 8, 16, 1, float("inf"), lo, hi, 16, 16, None, None) == rt.RETINA_EINVAL
    assert m(ctypes.byref(ev), 1, 0.5, 8, None, 1, 0.1, lo, hi, 16, 16, None, None) == rt.RETINA_EINVAL
    assert m(ctypes.byref(ev), 1, 0.5, 0, None, 1, 0.1, lo, hi, None, None, None, None) == rt.RETINA_OK


def test_newton_validation(L):
    for fn in (L.retina_multistart_newton, L.retina_multistart_newton_ex, L.retina_multistart_newton_ex2):
        ex = fn is not L.retina_multistart_newton
        ex2 = fn is L.retina_multistart_newton_ex2
        ev = _ev()
        lo, hi = _f(-1, -1), _f(1, 1)
        sg, et = _f(0.5, 0.2), _f(1e-3, 1e-3)

        def call(model=1, S=8, steps=2, sig=sg, eta=et, fs=0.2, mh=8, lo_=lo, hi_=hi, th=16, R=16):
            args = [ctypes.byref(ev), model, S, 16, steps, sig, eta, fs, mh, lo_, hi_, th, R, None]
            if ex:
                args.append(None)
            if ex2:
                args += [rt.MS_DENSE, None, ctypes.c_size_t(0), None]
            return fn(*args, None)

        assert call(model=0) == rt.RETINA_EUNSUPPORTED          # LINE2D has no Newton kernel
        assert call(model=9) == rt.RETINA_EINVAL
        assert call(S=-1) == rt.RETINA_EINVAL
        assert call(steps=-1) == rt.RETINA_EINVAL
        assert call(steps=17) == rt.RETINA_EUNSUPPORTED          # > kMaxNewtonSteps
        assert call(sig=_f(0.0, 0.2)) == rt.RETINA_EINVAL
        assert call(eta=_f(float("nan"), 1.0)) == rt.RETINA_EINVAL
        assert call(fs=-1.0) == rt.RETINA_EINVAL
        assert call(mh=-1) == rt.RETINA_EINVAL
        assert call(mh=127) == rt.RETINA_EUNSUPPORTED           # 2^-k formed exactly only for k <= 126
        assert call(lo_=hi, hi_=lo) == rt.RETINA_EINVAL
        assert call(th=None) == rt.RETINA_EINVAL
        assert call(S=0, th=None, R=None) == rt.RETINA_OK        # nothing to do


def test_newton_ex2_algorithm_and_workspace(L):
    """retina_multistart_newton_ex2: unknown algorithm, a missing or short workspace and too many
    seeds for the per-event sort are rejected before anything is launched; the workspace size is
    8 bytes per (event, seed) for RETINA_MS_CULLED (permutation + evaluation counts), 0 for dense."""
    f = L.retina_multistart_newton_ex2
    ev = _ev()
    lo, hi = _f(-1, -1), _f(1, 1)
    sg, et = _f(0.5, 0.2), _f(1e-3, 1e-3)

    def call(algo, S=8, ws=None, nbytes=0):
        return f(ctypes.byref(ev), 1, S, 16, 2, sg, et, 0.2, 8, lo, hi, 16, 16, None, None, algo, ws,
                 ctypes.c_size_t(nbytes), None, None)
    assert call(2) == rt.RETINA_EINVAL
    assert call(-1) == rt.RETINA_EINVAL
    assert call(rt.MS_CULLED) == rt.RETINA_EINVAL                            # no workspace
    assert call(rt.MS_CULLED, ws=16, nbytes=8) == rt.RETINA_EINVAL           # too small
    assert call(rt.MS_CULLED, S=16385, ws=16, nbytes=1 << 30) == rt.RETINA_EUNSUPPORTED
    wsz = L.retina_multistart_workspace_size
    assert wsz(3, 100, rt.MS_CULLED) == 3 * 100 * 8
    assert wsz(3, 100, rt.MS_DENSE) == 0 and wsz(0, 100, rt.MS_CULLED) == 0


def test_merge_validation(L):
    mg = L.retina_merge_tracks
    rad = _f(1e-3, 1e-3)
    args = (16, 16, rad, 5.0, 4, 16, 16, 16, 16, 16, None)
    assert mg(1, 16, 4, *args) == rt.RETINA_EINVAL
    assert mg(1, 16385, 2, *args) == rt.RETINA_EUNSUPPORTED
    assert mg(1, 16, 2, 16, 16, _f(-1.0, 1.0), 5.0, 4, 16, 16, 16, 16, 16, None) == rt.RETINA_EINVAL
    assert mg(0, 16, 2, *args) == rt.RETINA_OK


def test_product_package_never_touches_oracle():
    pkg = os.path.join(ROOT, "paper_1709_08610_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle/", ""), f
