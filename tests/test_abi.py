"""CPU checks of the C ABI: libpasa.so builds, loads, exports every symbol
include/pasa.h declares, and validates arguments on the host (no GPU calls)."""
import ctypes
import os
import re

import pytest

from paper_2604_12219_b200 import _C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2604_12219_b200 import build
    build.build()
    return _C.lib()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "pasa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(pasa_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_header_declarations_match_binding():
    assert declared_functions() == sorted(_C.EXPORTS)


def test_library_exports_every_declared_symbol(L):
    for name in declared_functions():
        assert hasattr(L, name), name
    assert b"sm_100a" in L.pasa_version()


def test_layer_seed_matches_splitmix_vectors(L):
    assert L.pasa_layer_seed(0, 0) == 0xE220A8397B1DCDAF
    assert L.pasa_layer_seed(42, 0) == 0xBDD732262FEB6E95


def test_library_has_tcgen05_and_tma_sass():
    """The tensor-core kernel is compiled to UTCHMMA/UTMALDG/LDTM (sm_100a), not HMMA."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump missing")
    sass = subprocess.run([exe, "-sass", _C.LIB_PATH], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM", "STTM", "UTCBAR"):
        assert mnem in sass, mnem


def cfg(**kw):
    d = dict(Bq=128, Bk=64, G=32, comp=0, beta=0.1, H_total=4, head_offset=0)
    d.update(kw)
    return _C.PasaRouteCfg(**d)


def test_route_workspace_validation(L):
    c = cfg()
    n = L.pasa_route_workspace_bytes(ctypes.byref(c), 1, 75600, 4, 128)
    assert n > 0
    for bad, why in [(cfg(Bk=32), "Bk"), (cfg(Bq=96), "Bq"), (cfg(G=0), "G"),
                     (cfg(beta=-1.0), "beta"), (cfg(head_offset=1), "H_total")]:
        assert L.pasa_route_workspace_bytes(ctypes.byref(bad), 1, 4096, 4, 128) == 0, why
        assert L.pasa_last_error()
    assert L.pasa_route_workspace_bytes(ctypes.byref(c), 1, 4096, 4, 96) == 0
    # N_K <= 4096 (S <= 262,144 at Bk = 64): the attention kernels' op-list capacity
    assert L.pasa_route_workspace_bytes(ctypes.byref(c), 1, 64 * 4096, 4, 128) > 0
    assert L.pasa_route_workspace_bytes(ctypes.byref(c), 1, 64 * 4097, 4, 128) == 0


def test_prior_workspace_validation(L):
    """Eq. 8 prior (NEXT 1): prior in {0,1,2}, eps > 0; the prior-enabled layout
    adds het + prior [BH][N_K] and fp64 group sums [BH][N_G][D][D] + Hbar [BH][D][D]."""
    S, H, D = 4096, 4, 128
    base = L.pasa_route_workspace_bytes(ctypes.byref(cfg()), 1, S, H, D)
    withp = L.pasa_route_workspace_bytes(ctypes.byref(cfg(prior=1, eps=1e-6)), 1, S, H, D)
    NK, NG = S // 64, (S // 64 + 31) // 32
    assert withp - base >= 8 * (2 * H * NK + H * NG * D * D + H * D * D)   # at least
    for bad in (cfg(prior=3, eps=1e-6), cfg(prior=1, eps=0.0), cfg(prior=2, eps=float("nan"))):
        assert L.pasa_route_workspace_bytes(ctypes.byref(bad), 1, S, H, D) == 0
        assert L.pasa_last_error()


def test_init_rejects_small_workspace_without_touching_device(L):
    c = cfg()
    n = L.pasa_route_workspace_bytes(ctypes.byref(c), 1, 4096, 4, 128)
    h = ctypes.c_void_p()
    fake = ctypes.c_void_p(0x10000)  # never dereferenced on the host
    assert L.pasa_route_init(fake, n - 1, ctypes.byref(c), 1, 4096, 4, 128,
                             ctypes.byref(h)) == _C.PASA_ENOSPACE
    assert L.pasa_route_init(fake, n, ctypes.byref(c), 1, 4096, 4, 128, ctypes.byref(h)) == 0
    dims = (ctypes.c_int64 * 7)()
    assert L.pasa_route_dims(h, dims) == 0
    assert list(dims) == [1, 4096, 4, 128, 32, 64, 2]
    L.pasa_route_fini(h)
    hb = ctypes.c_void_p()
    assert L.pasa_budget_init(fake, 8, ctypes.byref(hb)) == _C.PASA_ENOSPACE
    assert L.pasa_budget_init(fake, L.pasa_budget_workspace_bytes(), ctypes.byref(hb)) == 0
    L.pasa_budget_fini(hb)


def test_budget_host_validation(L):
    hb = ctypes.c_void_p()
    fake = ctypes.c_void_p(0x10000)
    assert L.pasa_budget_init(fake, L.pasa_budget_workspace_bytes(), ctypes.byref(hb)) == 0
    x = _C.PasaLatent(0x20000, 1, 0, 1024)
    sc = _C.PasaSchedule(50, 25, 0.15, 0.2, 0.0, 1.0, 1.0, 1.0, None, 0, 0)
    rc = L.pasa_budget(ctypes.byref(x), ctypes.byref(x), ctypes.byref(x), ctypes.byref(sc), hb, None)
    assert rc == _C.PASA_EDEGENERATE
    sc = _C.PasaSchedule(50, 50, 0.15, 0.2, 1.0, 1.0, 1.0, 1.0, None, 0, 0)
    assert L.pasa_budget(ctypes.byref(x), ctypes.byref(x), ctypes.byref(x), ctypes.byref(sc), hb,
                         None) == _C.PASA_EINVAL
    sc = _C.PasaSchedule(50, 20, 0.15, 0.2, 1.0, 0.0, 1.0, 1.0, None, 0, 0)
    assert L.pasa_budget(ctypes.byref(x), ctypes.byref(x), ctypes.byref(x), ctypes.byref(sc), hb,
                         None) == _C.PASA_EINVAL
    y = _C.PasaLatent(0x20000, 0, 0, 1024)  # bf16 vs fp32
    sc = _C.PasaSchedule(50, 20, 0.15, 0.2, 1.0, 1.0, 1.0, 1.0, None, 0, 0)
    assert L.pasa_budget(ctypes.byref(x), ctypes.byref(y), ctypes.byref(x), ctypes.byref(sc), hb,
                         None) == _C.PASA_EDTYPE
    L.pasa_budget_fini(hb)


def test_route_attn_host_validation(L):
    c = cfg(H_total=2)
    h = ctypes.c_void_p()
    fake = ctypes.c_void_p(0x10000)
    n = L.pasa_route_workspace_bytes(ctypes.byref(c), 1, 1000, 2, 64)
    assert L.pasa_route_init(fake, n, ctypes.byref(c), 1, 1000, 2, 64, ctypes.byref(h)) == 0
    hb = ctypes.c_void_p()
    assert L.pasa_budget_init(fake, L.pasa_budget_workspace_bytes(), ctypes.byref(hb)) == 0
    good = _C.PasaTensor(0x40000, 0, 0, 1, 1000, 2, 64, 1000 * 128, 128, 64)
    wrong_s = _C.PasaTensor(0x40000, 0, 0, 1, 999, 2, 64, 1000 * 128, 128, 64)
    wrong_dt = _C.PasaTensor(0x40000, 1, 0, 1, 1000, 2, 64, 1000 * 128, 128, 64)
    misalign = _C.PasaTensor(0x40002, 0, 0, 1, 1000, 2, 64, 1000 * 128, 128, 64)
    assert L.pasa_route(ctypes.byref(wrong_s), ctypes.byref(good), hb, 1, 3, h, None) == _C.PASA_ESHAPE
    assert L.pasa_route(ctypes.byref(good), ctypes.byref(wrong_dt), hb, 1, 3, h, None) == _C.PASA_EDTYPE
    assert L.pasa_route(ctypes.byref(misalign), ctypes.byref(good), hb, 1, 3, h, None) == _C.PASA_ESHAPE
    # attention before any route was built
    assert L.pasa_attn(ctypes.byref(good), ctypes.byref(good), ctypes.byref(good), h,
                       ctypes.byref(good), None) == _C.PASA_EINVAL
    L.pasa_route_fini(h)
    L.pasa_budget_fini(hb)


def test_zero_copy_host_validation(L):
    """pasa_route_zc / pasa_attn_zc reject bad shard tables on the host, launching nothing:
    NULL handles, a shard table whose starts do not cover [0, S), a head range outside the
    shards' H, fp32 shards, misaligned bases, and attention before a zero-copy route."""
    c = cfg(H_total=4)
    c.head_offset = 2
    h = ctypes.c_void_p()
    fake = ctypes.c_void_p(0x10000)
    n = L.pasa_route_workspace_bytes(ctypes.byref(c), 1, 1000, 2, 64)
    assert L.pasa_route_init(fake, n, ctypes.byref(c), 1, 1000, 2, 64, ctypes.byref(h)) == 0
    hb = ctypes.c_void_p()
    assert L.pasa_budget_init(fake, L.pasa_budget_workspace_bytes(), ctypes.byref(hb)) == 0
    loc = _C.PasaTensor(0x40000, 0, 0, 1, 1000, 2, 64, 1000 * 128, 128, 64)

    def shards(H=4, starts=(0, 400, 1000), dtype=0, base=0x80000):
        d = _C.PasaShards()
        d.dtype, d.nshards, d.S, d.H, d.D, d.sS, d.sH = dtype, len(starts) - 1, 1000, H, 64, H * 64, 64
        for i, s in enumerate(starts):
            d.start[i] = s
        for i in range(len(starts) - 1):
            d.data[i] = base + i * 0x100000
        return d

    good = shards()
    args = lambda q, hh=h, bb=hb: (ctypes.byref(q), ctypes.byref(good), ctypes.byref(good), bb, 1,  # noqa: E731
                                   3, hh, ctypes.byref(loc), ctypes.byref(loc), ctypes.byref(loc), None)
    assert L.pasa_route_zc(*args(good, hh=None)) == _C.PASA_EINVAL
    assert L.pasa_route_zc(*args(shards(starts=(0, 400, 999)))) == _C.PASA_EINVAL     # S not covered
    assert L.pasa_route_zc(*args(shards(starts=(0, 400, 400, 1000)))) == _C.PASA_EINVAL  # empty shard
    assert L.pasa_route_zc(*args(shards(H=3))) == _C.PASA_EINVAL                       # heads 2..3 of 3
    assert L.pasa_route_zc(*args(shards(dtype=1))) == _C.PASA_EDTYPE
    assert L.pasa_route_zc(*args(shards(base=0x80004))) == _C.PASA_EINVAL              # misaligned
    assert L.pasa_attn_zc(ctypes.byref(loc), ctypes.byref(loc), ctypes.byref(loc), h,
                          ctypes.byref(good), None) == _C.PASA_EINVAL   # no route built yet
    L.pasa_route_fini(h)
    L.pasa_budget_fini(hb)


def test_shards_desc_layout():
    """The Python shard table: starts accumulate the shard lengths, strides are checked."""
    import torch
    from paper_2604_12219_b200 import api
    xs = [torch.zeros(1, n, 3, 64, dtype=torch.bfloat16) for n in (5, 1, 10)]
    # tensor_desc needs CUDA; shards_desc only reads shapes, strides and data pointers
    d = api.shards_desc(xs)
    assert d.nshards == 3 and d.S == 16 and list(d.start[:4]) == [0, 5, 6, 16]
    assert d.sS == 3 * 64 and d.sH == 64
    with pytest.raises(ValueError):
        api.shards_desc([xs[0], torch.zeros(1, 4, 2, 64, dtype=torch.bfloat16)])
