"""NumPy fp64 brute force for tiny inputs -- TEST INFRASTRUCTURE ONLY.

An independent second reading of the same definitions as ``pasa_oracle.c``,
written in a different algebraic arrangement so that the two pin each other:

* dense attention is Eq. 1 with a full softmax;
* the piecewise output evaluates Eq. 7 per dropped block
  *inside* the block sum, ``sum_{j in U} alpha_tj [Vsum_j + s q_t C_j]`` with
  ``C_j`` the group mean of the per-block ``H_j`` (App. B), not the
  regrouped ``sum_g A_g q_t Hbar_g`` form the C oracle uses;
* the denominator counts each token of a dropped block with its centroid
  logit (reading R-2), i.e. the softmax over a length-S logit vector where
  dropped tokens carry their block's centroid logit;
* Philox4x32-10 is vectorised over counters with NumPy uint64 arithmetic;
* top-k uses ``np.lexsort`` instead of a comparator sort.
"""
from __future__ import annotations

import numpy as np

PHILOX_M = (0xD2511F53, 0xCD9E8D57)
PHILOX_W = (0x9E3779B9, 0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr: np.ndarray, key) -> np.ndarray:
    """ctr: [..., 4] uint32, key: (k0, k1).  Returns [..., 4] uint32."""
    c = [np.asarray(ctr[..., i], dtype=np.uint64) for i in range(4)]
    k0, k1 = np.uint64(key[0]), np.uint64(key[1])
    M0, M1 = np.uint64(PHILOX_M[0]), np.uint64(PHILOX_M[1])
    for r in range(10):
        if r:
            k0 = (k0 + np.uint64(PHILOX_W[0])) & MASK32
            k1 = (k1 + np.uint64(PHILOX_W[1])) & MASK32
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        c = [((p1 >> np.uint64(32)) ^ c[1] ^ k0) & MASK32, p1 & MASK32,
             ((p0 >> np.uint64(32)) ^ c[3] ^ k1) & MASK32, p0 & MASK32]
    return np.stack([x.astype(np.uint32) for x in c], axis=-1)


def gumbel_grid(seed: int, step: int, gh: int, NQ: int, NK: int) -> np.ndarray:
    """g[i, j] from word j mod 4 of counter (j // 4, i, gh, step), key (lo32 seed, hi32 seed)
    (reading R-11: one Philox4x32-10 call serves four consecutive blocks)."""
    i, j = np.meshgrid(np.arange(NQ), np.arange(NK), indexing="ij")
    ctr = np.stack([j // 4, i, np.full_like(i, gh), np.full_like(i, step)], -1).astype(np.uint32)
    words = philox4x32_10(ctr, (seed & 0xFFFFFFFF, seed >> 32))
    xw = np.take_along_axis(words, (j % 4)[..., None], axis=-1)[..., 0]
    u = (xw.astype(np.float64) + 0.5) * 2.0 ** -32
    return -np.log(-np.log(u))


def blocks(S: int, B: int):
    return [(j * B, min((j + 1) * B, S)) for j in range((S + B - 1) // B)]


def dense_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """One head, [S, D] each: softmax(q k^T / sqrt(D)) v (Eq. 1)."""
    s = 1.0 / np.sqrt(q.shape[1])
    L = s * (q @ k.T)
    L = L - L.max(axis=1, keepdims=True)
    P = np.exp(L)
    return (P / P.sum(axis=1, keepdims=True)) @ v


def route_head(q: np.ndarray, k: np.ndarray, Bq: int, Bk: int, kk: int, beta: float,
               seed: int, step: int, gh: int):
    """Returns (sel list of ascending arrays, rt scores [NQ, NK])."""
    S, D = q.shape
    Qb = np.stack([q[a:b].sum(0) / (b - a) for a, b in blocks(S, Bq)])
    Kb = np.stack([k[a:b].sum(0) / (b - a) for a, b in blocks(S, Bk)])
    r = (1.0 / np.sqrt(D)) * (Qb @ Kb.T)
    NQ, NK = r.shape
    if beta != 0.0:
        sig = r.std(axis=1, keepdims=True)
        r = r + (beta * sig) * gumbel_grid(seed, step, gh, NQ, NK)
    kk = max(1, min(kk, NK))
    sel = []
    for i in range(NQ):
        order = np.lexsort((np.arange(NK), -r[i]))  # primary: score desc, then j asc
        sel.append(np.sort(order[:kk]))
    return sel, r


def block_H(k: np.ndarray, v: np.ndarray, Bk: int) -> np.ndarray:
    """Eq. 5 per block: [NK, D, D]."""
    out = []
    for a, b in blocks(k.shape[0], Bk):
        kc = k[a:b] - k[a:b].mean(0, keepdims=True)
        out.append(np.einsum("na,nb->ab", kc, v[a:b]))
    return np.stack(out)


def piecewise(q, k, v, sel, Bq: int, Bk: int, G: int, comp: str = "grouped") -> np.ndarray:
    """Eq. 7 with grouped surrogate, evaluated directly per dropped block.  One head."""
    S, D = q.shape
    s = 1.0 / np.sqrt(D)
    kb = blocks(S, Bk)
    NK = len(kb)
    Kbar = np.stack([k[a:b].mean(0) for a, b in kb])
    Vsum = np.stack([v[a:b].sum(0) for a, b in kb])
    Hj = block_H(k, v, Bk)
    C = np.zeros_like(Hj)
    for g0 in range(0, NK, G):
        C[g0:g0 + G] = Hj[g0:g0 + G].mean(0)
    out = np.zeros_like(q)
    for i, (a, b) in enumerate(blocks(S, Bq)):
        chosen = np.zeros(NK, bool)
        chosen[sel[i]] = True
        for t in range(a, b):
            # per-token logit vector: exact for chosen tokens, centroid for dropped ones
            logit = np.full(S, -np.inf)
            for j, (u0, u1) in enumerate(kb):
                if chosen[j]:
                    logit[u0:u1] = s * (k[u0:u1] @ q[t])
                elif comp != "none":
                    logit[u0:u1] = s * (Kbar[j] @ q[t])
            m = logit.max()
            w = np.exp(logit - m)
            den = w.sum()
            num = np.zeros(D)
            for j, (u0, u1) in enumerate(kb):
                if chosen[j]:
                    num += w[u0:u1] @ v[u0:u1]
                elif comp != "none":
                    alpha = w[u0]
                    term = Vsum[j].copy()
                    if comp == "grouped":
                        term += s * (q[t] @ C[j])
                    num += alpha * term
            out[t] = num / den
    return out
