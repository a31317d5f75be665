"""PASA (arXiv 2604.12219) per-step sparse self-attention on B200 (sm_100a).

budget -> route -> attn through the C ABI of libpasa.so (include/pasa.h).
"""
from ._C import PasaError  # noqa: F401
from .api import (Budget, Route, RouteCfg, attn, attn_zc, last_launch_count, layer_seed,  # noqa: F401
                  route_zc)

__all__ = ["Budget", "Route", "RouteCfg", "attn", "attn_zc", "route_zc", "layer_seed",
           "last_launch_count", "PasaError"]
