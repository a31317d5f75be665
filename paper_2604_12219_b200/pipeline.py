"""Host-resident inputs: one PASA step with the PCIe transfers overlapped with
compute (CUDA streams, no tracing compiler).

A serving process often holds q, k, v (and the latents) in pinned host memory.
Copying everything, computing, then copying the output back serialises three
phases whose costs are comparable at video sizes (Wan 2.1-14B 720p: 2.3 GB in,
0.77 GB out, ~25 ms of compute).  Every (b, h) is independent,
so the heads are split into chunks:

    copy-in stream :  latents | q,k,v chunk 0 | chunk 1 | chunk 2 | ...
    compute stream :            budget | route+attn 0 | route+attn 1 | ...
    copy-out stream:                           out 0  |  out 1  | ...

Each chunk has its own route handle whose ``head_offset`` / ``H_total`` name
its global heads, so the Philox keying (R-11, R-20) -- and therefore the result
-- is bitwise identical to the single-shot call.  Strided head runs of the
[B, S, H, D] host tensors move with one ``pasa_copy2d`` (cudaMemcpy2DAsync) per
tensor and chunk.  Everything on the device runs in libpasa.so's kernels.
"""
from __future__ import annotations

import ctypes
from dataclasses import replace
from typing import Optional, Sequence

import torch

from . import _C
from .api import Budget, Route, RouteCfg, attn


def _copy2d(dst: int, dpitch: int, src: int, spitch: int, width: int, height: int, kind: int,
            stream: torch.cuda.Stream):
    _C.check(_C.lib().pasa_copy2d(ctypes.c_void_p(dst), dpitch, ctypes.c_void_p(src), spitch, width,
                                  height, kind, ctypes.c_void_p(stream.cuda_stream)),
             "pasa_copy2d")


class HostPipeline:
    """PASA budget + route + attention for pinned HOST q, k, v, out ([B, S, H, D],
    contiguous, bf16) split into ``n_chunks`` head chunks on three streams."""

    def __init__(self, B: int, S: int, H: int, D: int, cfg: Optional[RouteCfg] = None,
                 n_chunks: int = 8, device=None, dtype=torch.bfloat16, taper: bool = True,
                 attn_kw: Optional[dict] = None):
        self.shape = (B, S, H, D)
        self.attn_kw = dict(attn_kw or {})   # extra pasa_attn flags (e.g. cta_pair=True)
        self.dtype = dtype
        self.device = torch.device(device if device is not None else "cuda")
        cfg = cfg or RouteCfg()
        H_total = cfg.H_total if cfg.H_total is not None else H
        n_chunks = max(1, min(n_chunks, H))
        edges = [round(c * H / n_chunks) for c in range(n_chunks + 1)]
        self.chunks = [(a, b) for a, b in zip(edges[:-1], edges[1:]) if b > a]
        nq = -(-S // cfg.Bq)
        if (taper and len(self.chunks) > 1 and self.chunks[-1][1] - self.chunks[-1][0] > 1
                and nq >= 296):
            # the last chunk's compute and D2H copy run after every H2D copy (the drain):
            # split it into single heads so the drain is one head's work, when one head
            # still fills the GPU (>= 2 CTAs per SM; Wan-14B e2e 46.5 -> 45.6 ms)
            a, b = self.chunks.pop()
            self.chunks += [(h, h + 1) for h in range(a, b)]
        self.bufs, self.routes = [], []
        for a, b in self.chunks:
            hc = b - a
            t = lambda: torch.empty((B, S, hc, D), dtype=dtype, device=self.device)  # noqa: E731
            self.bufs.append((t(), t(), t(), t()))                      # q, k, v, out
            ccfg = replace(cfg, H_total=H_total, head_offset=cfg.head_offset + a)
            self.routes.append(Route(B, S, hc, D, ccfg, self.device))
        self.s_in = torch.cuda.Stream(self.device)
        self.s_cmp = torch.cuda.Stream(self.device)
        self.s_out = torch.cuda.Stream(self.device)
        self.budget = Budget(self.device)
        self._lat = None
        self.h2d_bytes = self.d2h_bytes = 0

    def _latent_bufs(self, latents: Sequence[torch.Tensor]):
        if self._lat is None or [t.shape for t in self._lat] != [t.shape for t in latents]:
            self._lat = [torch.empty(t.shape, dtype=t.dtype, device=self.device) for t in latents]
        return self._lat

    def __call__(self, hq: torch.Tensor, hk: torch.Tensor, hv: torch.Tensor, hout: torch.Tensor,
                 latents: Sequence[torch.Tensor], seed: int, step: int, *, v_for_prior=False,
                 **schedule):
        """Enqueue denoising step ``step``; returns the event recorded after the last
        D2H copy.  ``latents`` = (x_t, x_{t-1}, x_{t-2}) (or two velocities with
        kind="velocity") in pinned host memory; ``schedule`` = the other
        Budget.__call__ keywords (T, rho, l1_mean, h_t, h_tm1, rho_table, ...)."""
        B, S, H, D = self.shape
        for t in (hq, hk, hv, hout):
            if tuple(t.shape) != self.shape or not t.is_contiguous() or t.dtype != self.dtype:
                raise ValueError("host q/k/v/out must be contiguous [B, S, H, D] of the pipeline dtype")
            if not t.is_pinned():
                raise ValueError("host tensors must be pinned (torch.Tensor.pin_memory())")
        es = torch.tensor([], dtype=self.dtype).element_size()
        row = H * D * es                        # host row pitch (one token, all heads)
        cur = torch.cuda.current_stream(self.device)
        start = torch.cuda.Event()
        start.record(cur)
        for s in (self.s_in, self.s_cmp, self.s_out):
            s.wait_event(start)
        # latents, then the budget (once per step)
        dl = self._latent_bufs(latents)
        with torch.cuda.stream(self.s_in):
            for d, h in zip(dl, latents):
                d.copy_(h, non_blocking=True)
            ev_lat = torch.cuda.Event()
            ev_lat.record(self.s_in)
        self.s_cmp.wait_event(ev_lat)
        with torch.cuda.stream(self.s_cmp):
            xs = list(dl) + [None] * (3 - len(dl))
            self.budget(xs[0], xs[1], xs[2], step=step, stream=self.s_cmp, **schedule)
        h2d = sum(t.numel() * t.element_size() for t in latents)
        d2h = 0
        ev_in, ev_cmp = [], []
        for (a, b), (q, k, v, o) in zip(self.chunks, self.bufs):
            w = (b - a) * D * es
            for src, dst in ((hq, q), (hk, k), (hv, v)):
                _copy2d(dst.data_ptr(), w, src.data_ptr() + a * D * es, row, w, B * S, 1, self.s_in)
                h2d += w * B * S
            e = torch.cuda.Event()
            e.record(self.s_in)
            ev_in.append(e)
        for (a, b), (q, k, v, o), route, e in zip(self.chunks, self.bufs, self.routes, ev_in):
            self.s_cmp.wait_event(e)
            route(q, k, self.budget, seed, step, v=v if v_for_prior else None, stream=self.s_cmp)
            attn(q, k, v, route, o, stream=self.s_cmp, **self.attn_kw)
            ec = torch.cuda.Event()
            ec.record(self.s_cmp)
            ev_cmp.append(ec)
        for (a, b), (q, k, v, o), e in zip(self.chunks, self.bufs, ev_cmp):
            self.s_out.wait_event(e)
            w = (b - a) * D * es
            _copy2d(hout.data_ptr() + a * D * es, row, o.data_ptr(), w, w, B * S, 2, self.s_out)
            d2h += w * B * S
        done = torch.cuda.Event()
        done.record(self.s_out)
        cur.wait_event(done)
        self.h2d_bytes, self.d2h_bytes = h2d, d2h
        return done
