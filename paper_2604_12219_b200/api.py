"""Python face of libpasa.so: torch tensors in, C-ABI calls out.

PyTorch supplies device memory (workspaces via ``torch.empty``), the current
CUDA stream and nothing else; every arithmetic step runs in the library's
CUDA kernels.  Names follow include/pasa.h: ``Budget`` wraps
``pasa_budget``, ``Route`` wraps ``pasa_route``, ``attn`` wraps ``pasa_attn``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _C

_DT = {torch.bfloat16: _C.PASA_BF16, torch.float32: _C.PASA_F32}


def _stream_ptr(stream: Optional[torch.cuda.Stream] = None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def tensor_desc(x: torch.Tensor) -> _C.PasaTensor:
    """[B, S, H, D] CUDA tensor (D contiguous) -> pasa_tensor."""
    if x.dim() != 4:
        raise ValueError(f"expected [B, S, H, D], got shape {tuple(x.shape)}")
    if not x.is_cuda:
        raise ValueError("pasa tensors must live on a CUDA device")
    if x.dtype not in _DT:
        raise TypeError(f"dtype {x.dtype} not supported (bf16 or fp32)")
    if x.stride(3) != 1:
        raise ValueError("the head dimension D must be contiguous")
    B, S, H, D = x.shape
    return _C.PasaTensor(x.data_ptr(), _DT[x.dtype], 0, B, S, H, D, x.stride(0), x.stride(1),
                         x.stride(2))


def latent_desc(x: torch.Tensor) -> _C.PasaLatent:
    if not x.is_cuda or not x.is_contiguous():
        raise ValueError("latents must be contiguous CUDA tensors")
    if x.dtype not in _DT:
        raise TypeError(f"latent dtype {x.dtype} not supported")
    return _C.PasaLatent(x.data_ptr(), _DT[x.dtype], 0, x.numel())


def layer_seed(seed: int, layer: int) -> int:
    """Per-layer Philox key (reading R-11): pasa_layer_seed(seed, layer)."""
    return int(_C.lib().pasa_layer_seed(seed, layer))


def last_launch_count() -> int:
    return int(_C.lib().pasa_last_launch_count())


class Budget:
    """Device-resident budget record {l1, alpha, rho_t, dense, clipped} (Eqs. 9-11)."""

    def __init__(self, device=None):
        L = _C.lib()
        self.device = torch.device(device if device is not None else "cuda")
        n = L.pasa_budget_workspace_bytes()
        self.ws = torch.empty(n, dtype=torch.uint8, device=self.device)
        h = ctypes.c_void_p()
        _C.check(L.pasa_budget_init(ctypes.c_void_p(self.ws.data_ptr()), n, ctypes.byref(h)),
                 "pasa_budget_init")
        self.handle = h

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _C.lib().pasa_budget_fini(self.handle)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass

    def _schedule(self, T, step, rho, dense_frac, l1_mean, h_t, h_tm1, rho_max, rho_table, kind):
        kind_i = _C.PASA_IN_VELOCITY if kind == "velocity" else _C.PASA_IN_LATENT
        tab = None
        if rho_table is not None:
            if len(rho_table) < T:
                raise ValueError(f"rho_table has {len(rho_table)} entries, needs T = {T}")
            self._tab = np.ascontiguousarray(np.asarray(rho_table, dtype=np.float64))
            tab = self._tab.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        return _C.PasaSchedule(T, step, rho, dense_frac, l1_mean, h_t, h_tm1, rho_max, tab, kind_i,
                               0)

    def __call__(self, x_t, x_tm1, x_tm2=None, *, T=50, step=25, rho=0.15, dense_frac=0.2,
                 l1_mean=1.0, h_t=1.0, h_tm1=1.0, rho_max=1.0, rho_table=None, kind="latent",
                 stream=None):
        a, b = latent_desc(x_t), latent_desc(x_tm1)
        c = latent_desc(x_tm2) if x_tm2 is not None else None
        sc = self._schedule(T, step, rho, dense_frac, l1_mean, h_t, h_tm1, rho_max, rho_table, kind)
        st = _C.lib().pasa_budget(ctypes.byref(a), ctypes.byref(b),
                                  ctypes.byref(c) if c is not None else None, ctypes.byref(sc),
                                  self.handle, _stream_ptr(stream))
        _C.check(st, "pasa_budget")
        return self

    def local_sum(self, x_t, x_tm1, x_tm2=None, out=None, *, T=50, step=25, rho=0.15,
                  dense_frac=0.2, l1_mean=1.0, h_t=1.0, h_tm1=1.0, rho_max=1.0, rho_table=None,
                  kind="latent", stream=None) -> torch.Tensor:
        """pasa_budget_local_sum: this rank's fp64 sum of |dv| (a 1-element device tensor)
        for latents sharded across ranks."""
        if out is None:
            out = torch.empty(1, dtype=torch.float64, device=x_t.device)
        a, b = latent_desc(x_t), latent_desc(x_tm1)
        c = latent_desc(x_tm2) if x_tm2 is not None else None
        sc = self._schedule(T, step, rho, dense_frac, l1_mean, h_t, h_tm1, rho_max, rho_table, kind)
        _C.check(_C.lib().pasa_budget_local_sum(
            ctypes.byref(a), ctypes.byref(b), ctypes.byref(c) if c is not None else None,
            ctypes.byref(sc), self.handle, ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)),
            "pasa_budget_local_sum")
        return out

    def from_sums(self, sums: torch.Tensor, n_total: int, *, T=50, step=25, rho=0.15,
                  dense_frac=0.2, l1_mean=1.0, h_t=1.0, h_tm1=1.0, rho_max=1.0, rho_table=None,
                  kind="latent", stream=None):
        """pasa_budget_from_sums: l = (sums in rank order) / n_total, then Eqs. 10-11."""
        if sums.dtype != torch.float64 or not sums.is_cuda or not sums.is_contiguous():
            raise ValueError("sums must be a contiguous float64 CUDA tensor")
        sc = self._schedule(T, step, rho, dense_frac, l1_mean, h_t, h_tm1, rho_max, rho_table, kind)
        _C.check(_C.lib().pasa_budget_from_sums(ctypes.c_void_p(sums.data_ptr()), sums.numel(),
                                                n_total, ctypes.byref(sc), self.handle,
                                                _stream_ptr(stream)), "pasa_budget_from_sums")
        return self

    def read(self, stream=None) -> dict:
        out = (ctypes.c_double * 5)()
        _C.check(_C.lib().pasa_budget_read(self.handle, out, _stream_ptr(stream)),
                 "pasa_budget_read")
        return dict(l1=out[0], alpha=out[1], rho_t=out[2], dense=bool(out[3]),
                    clipped=bool(out[4]))


@dataclass
class RouteCfg:
    Bq: int = 128
    Bk: int = 64
    G: int = 32
    comp: str = "grouped"
    beta: float = 0.1
    H_total: Optional[int] = None
    head_offset: int = 0
    prior: str = "none"          # Eq. 8 heterogeneity prior: "none" | "global" | "group"
    eps: float = 1e-6
    qb_begin: int = 0            # query blocks [qb_begin, qb_end) only; (0, 0) = all
    qb_end: int = 0              # (flattened (head, q-block) partition)
    qk_precision: str = "bf16"   # "fp8": opt-in FP8 QK^T variant (NEXT 4, R-30; own tolerance)

    def to_c(self, H: int) -> _C.PasaRouteCfg:
        return _C.PasaRouteCfg(self.Bq, self.Bk, self.G, _C.COMP[self.comp], self.beta,
                               self.H_total if self.H_total is not None else H, self.head_offset,
                               _C.PRIOR[self.prior], 0, self.eps, self.qb_begin, self.qb_end,
                               {"bf16": 0, "fp8": 1}[self.qk_precision], 0)


class Route:
    """Route workspace + handle for [B, S, H, D] activations (pasa_route_init)."""

    def __init__(self, B, S, H, D, cfg: Optional[RouteCfg] = None, device=None):
        L = _C.lib()
        self.cfg = cfg or RouteCfg()
        self.shape = (B, S, H, D)
        self.device = torch.device(device if device is not None else "cuda")
        c = self.cfg.to_c(H)
        self._c = c
        n = L.pasa_route_workspace_bytes(ctypes.byref(c), B, S, H, D)
        if n == 0:
            raise _C.PasaError(_C.PASA_EINVAL, "pasa_route_workspace_bytes",
                               L.pasa_last_error().decode())
        self.ws = torch.empty(n, dtype=torch.uint8, device=self.device)
        h = ctypes.c_void_p()
        _C.check(L.pasa_route_init(ctypes.c_void_p(self.ws.data_ptr()), n, ctypes.byref(c), B, S,
                                   H, D, ctypes.byref(h)), "pasa_route_init")
        self.handle = h
        dims = (ctypes.c_int64 * 7)()
        _C.check(L.pasa_route_dims(h, dims), "pasa_route_dims")
        self.NQ, self.NK, self.NG = dims[4], dims[5], dims[6]
        self.W = (self.NK + 31) // 32

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _C.lib().pasa_route_fini(self.handle)
        except Exception:  # pragma: no cover
            pass

    def __call__(self, q, k, budget: Budget, seed: int, step: int, v=None, stream=None):
        """pasa_route, or pasa_route_v when v is given (Eq. 8 prior enabled in cfg)."""
        qd, kd = tensor_desc(q), tensor_desc(k)
        if v is None:
            _C.check(_C.lib().pasa_route(ctypes.byref(qd), ctypes.byref(kd), budget.handle, seed,
                                         step, self.handle, _stream_ptr(stream)), "pasa_route")
        else:
            vd = tensor_desc(v)
            _C.check(_C.lib().pasa_route_v(ctypes.byref(qd), ctypes.byref(kd), ctypes.byref(vd),
                                           budget.handle, seed, step, self.handle,
                                           _stream_ptr(stream)), "pasa_route_v")
        return self

    def het(self, stream=None) -> np.ndarray:
        """||H_j - C||_F of the last pasa_route_v: float64 [B*H, N_K]."""
        B, S, H, D = self.shape
        out = np.zeros((B * H, self.NK))
        _C.check(_C.lib().pasa_route_het_read(self.handle, ctypes.c_void_p(out.ctypes.data),
                                              _stream_ptr(stream)), "pasa_route_het_read")
        return out

    def read(self, stream=None) -> dict:
        B, S, H, D = self.shape
        BH = B * H
        k = np.zeros(1, np.int32)
        idx = np.zeros((BH, self.NQ, self.NK), np.int32)
        cnt = np.zeros((BH, self.NQ), np.int32)
        mask = np.zeros((BH, self.NQ, self.W), np.uint32)
        P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
        _C.check(_C.lib().pasa_route_read(self.handle, P(k), P(idx), P(cnt), P(mask),
                                          _stream_ptr(stream)), "pasa_route_read")
        return dict(k=int(k[0]), idx=idx, count=cnt, mask=mask)

    def stats(self, stream=None):
        """Statistics of the last pasa_attn: (kbar, vsum, ht) as float64 numpy arrays,
        ht[bh, g, n, k] = Hbar^(g)[k][n].  Stored in that call's I/O dtype, which the
        binding recorded (pasa_attn_stats_read rejects a mismatched declaration)."""
        B, S, H, D = self.shape
        dtype = getattr(self, "_stats_dtype", None)
        if dtype is None:
            raise _C.PasaError(_C.PASA_EINVAL, "Route.stats", "no pasa_attn has run on this route")
        t = torch.empty
        kb = t((B * H, self.NK, D), dtype=dtype)
        vs = t((B * H, self.NK, D), dtype=dtype)
        ht = t((B * H, self.NG, D, D), dtype=dtype)
        _C.check(_C.lib().pasa_attn_stats_read(self.handle, ctypes.c_void_p(kb.data_ptr()),
                                               ctypes.c_void_p(vs.data_ptr()),
                                               ctypes.c_void_p(ht.data_ptr()), _DT[dtype],
                                               _stream_ptr(stream)), "pasa_attn_stats_read")
        return (kb.double().numpy(), vs.double().numpy(), ht.double().numpy())

    def pooled(self, stream=None):
        B, S, H, D = self.shape
        qb = np.zeros((B * H, self.NQ, D))
        kb = np.zeros((B * H, self.NK, D))
        _C.check(_C.lib().pasa_route_pooled_read(self.handle, ctypes.c_void_p(qb.ctypes.data),
                                                 ctypes.c_void_p(kb.ctypes.data),
                                                 _stream_ptr(stream)), "pasa_route_pooled_read")
        return qb, kb


def attn(q, k, v, route: Route, out=None, *, force_simt=False, stats_only=False,
         reuse_stats=False, cta_pair=False, stream=None):
    """pasa_attn: returns out ([B, S, H, D], q's dtype).  stats_only / reuse_stats
    split the call into its statistics and attention kernels; cta_pair runs a Bq = 256
    route on the tcgen05 cta_group::2 kernel (PASA_ATTN_* flags)."""
    if out is None:
        out = torch.empty_like(q)
    qd, kd, vd, od = tensor_desc(q), tensor_desc(k), tensor_desc(v), tensor_desc(out)
    flags = ((_C.PASA_ATTN_FORCE_SIMT if force_simt else 0)
             | (_C.PASA_ATTN_STATS_ONLY if stats_only else 0)
             | (_C.PASA_ATTN_REUSE_STATS if reuse_stats else 0)
             | (_C.PASA_ATTN_CTA_PAIR if cta_pair else 0))
    _C.check(_C.lib().pasa_attn_ex(ctypes.byref(qd), ctypes.byref(kd), ctypes.byref(vd),
                                   route.handle, ctypes.byref(od), flags, _stream_ptr(stream)),
             "pasa_attn")
    if not reuse_stats:
        route._stats_dtype = q.dtype   # the statistics pass ran in q's dtype
    return out


def shards_desc(shards) -> _C.PasaShards:
    """A list of P sequence shards [1, S_r, H, D] (bf16, CUDA, same strides; addressable
    from this process: local, peer or IPC-mapped) -> pasa_shards of the [1, S, H, D] whole."""
    if not 1 <= len(shards) <= 8:
        raise ValueError("1..8 shards")
    H, D = shards[0].shape[2], shards[0].shape[3]
    sS, sH = shards[0].stride(1), shards[0].stride(2)
    d = _C.PasaShards()
    d.dtype, d.nshards, d.H, d.D, d.sS, d.sH = _C.PASA_BF16, len(shards), H, D, sS, sH
    t = 0
    for r, x in enumerate(shards):
        if (x.dim() != 4 or x.shape[0] != 1 or x.shape[2:] != (H, D) or x.dtype != torch.bfloat16
                or x.stride(1) != sS or x.stride(2) != sH or x.stride(3) != 1):
            raise ValueError(f"shard {r}: expected [1, S_r, {H}, {D}] bf16 with the same strides")
        d.start[r] = t
        d.data[r] = x.data_ptr()
        t += x.shape[1]
    d.start[len(shards)] = t
    d.S = t
    return d


def route_zc(route: Route, q_shards, k_shards, v_shards, budget: Budget, seed: int, step: int,
             q_loc, k_loc, v_loc, stream=None):
    """pasa_route_zc: gather this rank's heads (route.cfg.head_offset ..) of q, k, v from every
    sequence shard into the local [1, S, Hl, D] buffers, pooling q and k in the same pass,
    then the fused score / bias / top-k kernel (include/pasa.h)."""
    qs, ks, vs = shards_desc(q_shards), shards_desc(k_shards), shards_desc(v_shards)
    ql, kl, vl = tensor_desc(q_loc), tensor_desc(k_loc), tensor_desc(v_loc)
    _C.check(_C.lib().pasa_route_zc(ctypes.byref(qs), ctypes.byref(ks), ctypes.byref(vs),
                                    budget.handle, seed, step, route.handle, ctypes.byref(ql),
                                    ctypes.byref(kl), ctypes.byref(vl), _stream_ptr(stream)),
             "pasa_route_zc")


def attn_zc(q_loc, k_loc, v_loc, route: Route, out_shards, stream=None):
    """pasa_attn_zc: statistics + attention over the local buffers, each output row stored
    straight into the shard (of out_shards) that owns its token."""
    ql, kl, vl = tensor_desc(q_loc), tensor_desc(k_loc), tensor_desc(v_loc)
    os_ = shards_desc(out_shards)
    _C.check(_C.lib().pasa_attn_zc(ctypes.byref(ql), ctypes.byref(kl), ctypes.byref(vl),
                                   route.handle, ctypes.byref(os_), _stream_ptr(stream)),
             "pasa_attn_zc")
    route._stats_dtype = torch.bfloat16
