"""fp64 CPU oracle for PASA (arXiv 2604.12219) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
``paper_2604_12219_b200`` never imports it, and nothing here imports the
product package: the two share no code (only ``synth/``'s seeded input
generators serve both).

The arithmetic lives in ``pasa_oracle.c`` (plain C, fp64, -ffp-contract=off);
this module only compiles it with gcc, converts arrays to float64 and
marshals pointers.  ``brute.py`` is an independent NumPy twin for tiny inputs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pasa_oracle.c")
_HDR = os.path.join(_HERE, "pasa_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

COMP = {"grouped": 0, "zeroth": 1, "none": 2}

GCC_FLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (building the checker is not using it)."""
    with _lock:
        stale = (not os.path.exists(_LIB)) or force or max(
            os.path.getmtime(_SRC), os.path.getmtime(_HDR)) > os.path.getmtime(_LIB)
        if stale:
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", *GCC_FLAGS, _SRC, "-o", tmp, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        D, I64, I32, U64, P = (ctypes.c_double, ctypes.c_int64, ctypes.c_int32,
                               ctypes.c_uint64, ctypes.c_void_p)
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_layer_seed.argtypes = [U64, I32]
        L.orc_layer_seed.restype = U64
        L.orc_gumbel.argtypes = [U64, I32, I64, I64, I64]
        L.orc_gumbel.restype = D
        L.orc_budget.argtypes = [P, P, P, I64, ctypes.c_int, D, D, I32, I32, D, D, D, D, P, P]
        L.orc_budget.restype = ctypes.c_int
        L.orc_l1.argtypes = [P, P, P, I64, ctypes.c_int, D, D]
        L.orc_l1.restype = D
        L.orc_density_to_k.argtypes = [D, I64]
        L.orc_density_to_k.restype = I64
        L.orc_route.argtypes = [P, P, I64, I64, I64, I64, I32, I32, D, U64, I32, I64, I64, I64,
                                P, P, P, P, D]
        L.orc_heterogeneity.argtypes = [P, P, I64, I64, I32, I32, I32, P]
        L.orc_calibrate.argtypes = [P, I32, I32, D, D, D, P, P, P, P]
        L.orc_calibrate.restype = ctypes.c_int
        L.orc_block_means.argtypes = [P, I64, I64, I32, P]
        L.orc_block_stats.argtypes = [P, P, I64, I64, I32, I32, P, P, P, P]
        L.orc_attn_with_route.argtypes = [P, P, P, I64, I64, I64, I32, I32, I32, I32, P, P, I64, P]
        L.orc_attn_pairs.argtypes = [P, P, P, I64, I64, I64, I32, I32, I32, I32, P, P, I64, P,
                                     I64, P]
        L.orc_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def f64(x) -> np.ndarray:
    """Exact upcast of the values the GPU receives (torch bf16/f32 or numpy)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return np.ascontiguousarray(x.detach().to("cpu").to(torch.float64).numpy())
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def heads(x) -> np.ndarray:
    """[B, S, H, D] -> contiguous fp64 [B*H, S, D] (per-head slices)."""
    a = f64(x)
    B, S, H, D = a.shape
    return np.ascontiguousarray(a.transpose(0, 2, 1, 3)).reshape(B * H, S, D)


def unheads(a: np.ndarray, B: int, H: int) -> np.ndarray:
    BH, S, D = a.shape
    return np.ascontiguousarray(a.reshape(B, H, S, D).transpose(0, 2, 1, 3))


def num_threads() -> int:
    return int(lib().orc_num_threads())


# ---------------------------------------------------------------------------
def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32).copy()
    k = np.asarray(key, dtype=np.uint32).copy()
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def layer_seed(seed: int, layer: int) -> int:
    return int(lib().orc_layer_seed(seed, layer))


def gumbel(seed: int, step: int, gh: int, i: int, j: int) -> float:
    return float(lib().orc_gumbel(seed, step, gh, i, j))


def density_to_k(rho_t: float, n_blocks: int) -> int:
    return int(lib().orc_density_to_k(rho_t, n_blocks))


def l1(x_t, x_tm1, x_tm2=None, kind: int = 0, h_t: float = 1.0, h_tm1: float = 1.0) -> float:
    a, b = f64(x_t).ravel(), f64(x_tm1).ravel()
    c = f64(x_tm2).ravel() if x_tm2 is not None else b
    return float(lib().orc_l1(_ptr(a), _ptr(b), _ptr(c), a.size, kind, h_t, h_tm1))


def budget(x_t, x_tm1, x_tm2=None, *, kind=0, h_t=1.0, h_tm1=1.0, T=50, step=25, rho=0.15,
           dense_frac=0.2, l1_mean=1.0, rho_max=1.0, rho_table=None):
    """Returns dict(l1, alpha, rho_t, dense, clipped) or raises ValueError."""
    a, b = f64(x_t).ravel(), f64(x_tm1).ravel()
    c = f64(x_tm2).ravel() if x_tm2 is not None else b
    out = np.zeros(5)
    tab = None if rho_table is None else f64(rho_table).ravel()
    rc = lib().orc_budget(_ptr(a), _ptr(b), _ptr(c), a.size, kind, h_t, h_tm1, T, step, rho,
                          dense_frac, l1_mean, rho_max, None if tab is None else _ptr(tab),
                          _ptr(out))
    if rc != 0:
        raise ValueError("oracle budget rejected its input")
    return dict(l1=out[0], alpha=out[1], rho_t=out[2], dense=bool(out[3]), clipped=bool(out[4]))


def block_means(x_head, Bsz: int) -> np.ndarray:
    x = f64(x_head)
    S, D = x.shape
    nb = (S + Bsz - 1) // Bsz
    out = np.zeros((nb, D))
    lib().orc_block_means(_ptr(x), S, D, Bsz, _ptr(out))
    return out


def route(q, k, *, Bq=64, Bk=64, beta=0.1, seed=42, step=25, H_total=None, head_offset=0,
          rho_t=None, kk=None, want_scores=False, het=None, eps=1e-6):
    """q, k: [B, S, H, D] (torch or numpy).  Returns dict(idx [B*H, N_Q, kk] int32,
    mask [B*H, N_Q, W] uint32, kk, scores?).  het: optional [B*H, N_K] norms of
    Eq. 8's prior (see heterogeneity); r_ij += log(het_j + eps)."""
    qa, ka = f64(q), f64(k)
    B, S, H, D = qa.shape
    qh, kh = heads(qa), heads(ka)
    NQ, NK = (S + Bq - 1) // Bq, (S + Bk - 1) // Bk
    if kk is None:
        kk = density_to_k(1.0 if rho_t is None else rho_t, NK)
    kk = max(1, min(int(kk), NK))
    W = (NK + 31) // 32
    idx = np.zeros((B * H, NQ, kk), dtype=np.int32)
    mask = np.zeros((B * H, NQ, W), dtype=np.uint32)
    scores = np.zeros((B * H, NQ, NK)) if want_scores else None
    lib().orc_route(_ptr(qh), _ptr(kh), B, H, S, D, Bq, Bk, beta, seed, step,
                    H if H_total is None else H_total, head_offset, kk, _ptr(idx), _ptr(mask),
                    None if scores is None else _ptr(scores), _het_ptr(het, B * H, NK), eps)
    out = dict(idx=idx, mask=mask, kk=kk)
    if want_scores:
        out["scores"] = scores
    return out


def calibrate(curves, *, rho=0.15, dense_frac=0.2, rho_max=1.0):
    """Offline Eqs. 9-11 from l-curves [N, T] (orc_calibrate).  Returns
    dict(rho_table, alpha, clipped, l1_mean) or raises ValueError."""
    c = np.ascontiguousarray(np.atleast_2d(np.asarray(curves, dtype=np.float64)))
    N, T = c.shape
    tab, alpha, lbar = np.zeros(T), np.zeros(T), np.zeros(1)
    clipped = np.zeros(T, dtype=np.int32)
    rc = lib().orc_calibrate(_ptr(c), N, T, rho, dense_frac, rho_max, _ptr(tab), _ptr(alpha),
                             _ptr(clipped), _ptr(lbar))
    if rc != 0:
        raise ValueError("orc_calibrate rejected the input")
    return dict(rho_table=tab, alpha=alpha, clipped=clipped.astype(bool), l1_mean=float(lbar[0]))


_HET_KEEP = []


def _het_ptr(het, BH, NK):
    if het is None:
        return None
    h = np.ascontiguousarray(np.asarray(het, dtype=np.float64))
    if h.shape != (BH, NK):
        raise ValueError(f"het must be [{BH}, {NK}], got {h.shape}")
    _HET_KEEP[:] = [h]
    return _ptr(h)


PRIOR = {"global": 1, "group": 2}


def heterogeneity(k_head, v_head, *, Bk=64, G=32, mode="global"):
    """Eq. 8 prior statistic for one head ([S, D] each): het[j] = ||H_j - C||_F,
    C = global Hbar (mode "global") or the group mean Hbar^(g(j)) ("group")."""
    k, v = f64(k_head), f64(v_head)
    S, D = k.shape
    NK = (S + Bk - 1) // Bk
    het = np.zeros(NK)
    lib().orc_heterogeneity(_ptr(k), _ptr(v), S, D, Bk, G, PRIOR[mode], _ptr(het))
    return het


def block_stats(k_head, v_head, *, Bk=64, G=32, want_blocks=False):
    """One head, [S, D] each.  Returns dict(Kbar, Vsum, Hbar[, H])."""
    k, v = f64(k_head), f64(v_head)
    S, D = k.shape
    NK = (S + Bk - 1) // Bk
    NG = (NK + G - 1) // G
    Kbar, Vsum = np.zeros((NK, D)), np.zeros((NK, D))
    Hbar = np.zeros((NG, D, D))
    Hblk = np.zeros((NK, D, D)) if want_blocks else None
    lib().orc_block_stats(_ptr(k), _ptr(v), S, D, Bk, G, _ptr(Kbar), _ptr(Vsum),
                          None if Hblk is None else _ptr(Hblk), _ptr(Hbar))
    out = dict(Kbar=Kbar, Vsum=Vsum, Hbar=Hbar)
    if want_blocks:
        out["H"] = Hblk
    return out


def attn_with_route(q, k, v, idx, count=None, *, Bq=64, Bk=64, G=32, comp="grouped"):
    """q, k, v: [B, S, H, D]; idx [B*H, N_Q, kk_stride] int32 (first count entries valid).
    Returns fp64 [B, S, H, D]."""
    qa = f64(q)
    B, S, H, D = qa.shape
    qh, kh, vh = heads(qa), heads(k), heads(v)
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int32))
    BH, NQ, kks = idx.shape
    if count is None:
        count = np.full((BH, NQ), kks, dtype=np.int32)
    count = np.ascontiguousarray(np.asarray(count, dtype=np.int32))
    out = np.zeros((BH, S, D))
    lib().orc_attn_with_route(_ptr(qh), _ptr(kh), _ptr(vh), BH, S, D, Bq, Bk, G, COMP[comp],
                              _ptr(idx), _ptr(count), kks, _ptr(out))
    return unheads(out, B, H)


def attn_pairs(q, k, v, idx, count, pairs, *, Bq=128, Bk=64, G=32, comp="grouped",
               qh=None, kh=None, vh=None):
    """Sampled attention: pairs = [(bh, i), ...].  Returns fp64 [npairs, Bq, D]
    (rows past S are zero).  qh/kh/vh: optional pre-converted [BH, S, D] fp64."""
    if qh is None:
        qh, kh, vh = heads(q), heads(k), heads(v)
    BH, S, D = qh.shape
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int32))
    count = np.ascontiguousarray(np.asarray(count, dtype=np.int32))
    kks = idx.shape[-1]
    pr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))
    out = np.zeros((pr.shape[0], Bq, D))
    lib().orc_attn_pairs(_ptr(qh), _ptr(kh), _ptr(vh), BH, S, D, Bq, Bk, G, COMP[comp],
                         _ptr(idx), _ptr(count), kks, _ptr(pr), pr.shape[0], _ptr(out))
    return out
