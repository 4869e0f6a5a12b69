"""Positional encoding (reference) and multiresolution hash-grid encoding (builder-defined).

``hann_band_weights`` / ``posenc`` / ``posenc_bwd`` restate ``ad:574-611``: band
weights ``w_k = (1 - cos(pi*clamp(alpha-k,0,1)))/2``, frequencies ``2^k pi``; columns are
raw xyz, then per band ``k`` the weighted ``sin`` xyz triple and ``cos`` xyz triple.

Hash grid -- PARITY UNPINNED (absent from the reference, SPEC non-goal ``S:139``):
* ``L`` levels, ``F = 2`` features, table size ``T = 2^log2_T`` per level;
* growth ``b = exp(ln(max_res/base_res)/(L-1))``, resolution ``N_l = floor(base_res*b^l + 1e-9)``;
* level ``l`` has vertices ``0..N_l`` per axis; it is dense (``idx = x + y(N+1) + z(N+1)^2``)
  when ``(N_l+1)^3 <= T`` else hashed
  (``idx = (x*1 ^ y*2654435761 ^ z*805459861) mod T``, uint32 arithmetic);
  level ``l`` occupies ``min((N_l+1)^3, T)`` consecutive table entries starting at a
  multiple of 4 (16-byte aligned in fp16, so a cell's two x-corners share one aligned
  4-entry block 3/4 of the time);
* a canonical point is normalised ``xn = clamp((x - cmin) * cinv, 0, 1)`` (float32, two
  rounded ops), ``pos = xn * N_l``, ``i0 = min(floor(pos), N_l - 1)``, ``f = pos - i0``;
* feature ``l`` = trilinear blend of the 8 corner entries accumulated in (a,b,c) order
  with weight ``(wx[a]*wy[b])*wz[c]``; output columns ``[l0f0, l0f1, l1f0, ...]``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

F32 = np.float32
U32 = np.uint32
PRIME_Y = 2654435761
PRIME_Z = 805459861


def hann_band_weights(num_bands, alpha, dtype=np.float64):
    k = np.arange(num_bands, dtype=dtype)
    x = np.clip(alpha - k, 0.0, 1.0)
    return ((1.0 - np.cos(np.pi * x)) / 2.0).astype(dtype)


def posenc(p, num_bands, alpha, dtype=np.float32):
    """(N,3) -> (N, 3+6L) with raw columns first (ad:581-600)."""
    dt = np.dtype(dtype).type
    x = np.asarray(p, dtype=dt)
    freqs = ((2.0 ** np.arange(num_bands, dtype=dt)) * dt(np.pi)).astype(dt)
    w = hann_band_weights(num_bands, alpha, dtype=dt)
    ang = (x[:, :, None] * freqs[None, None, :]).astype(dt)
    s, c = np.sin(ang), np.cos(ang)
    cols = [x]
    for k in range(num_bands):
        cols.append((w[k] * s[:, :, k]).astype(dt))
        cols.append((w[k] * c[:, :, k]).astype(dt))
    return np.concatenate(cols, axis=1)


def posenc_bwd(p, num_bands, alpha, g):
    """Gradient w.r.t. the raw points (ad:602-609)."""
    x = np.asarray(p, dtype=np.float64)
    d = x.shape[1]
    freqs = (2.0 ** np.arange(num_bands)) * np.pi
    w = hann_band_weights(num_bands, alpha)
    ang = x[:, :, None] * freqs[None, None, :]
    s, c = np.sin(ang), np.cos(ang)
    gp = g[:, :d].astype(np.float64).copy()
    for k in range(num_bands):
        gs = g[:, d + 2 * k * d: d + (2 * k + 1) * d]
        gc = g[:, d + (2 * k + 1) * d: d + (2 * k + 2) * d]
        gp += (w[k] * freqs[k]) * (gs * c[:, :, k] - gc * s[:, :, k])
    return gp


# ---------------------------------------------------------------------------
# Hash grid

@dataclass(frozen=True)
class HashGridSpec:
    n_levels: int = 16
    n_feat: int = 2
    log2_T: int = 14
    base_res: int = 16
    max_res: int = 512

    @property
    def table_size(self) -> int:
        return 1 << self.log2_T

    def resolutions(self):
        b = np.exp(np.log(self.max_res / self.base_res) / (self.n_levels - 1))
        return [int(np.floor(self.base_res * b ** l + 1e-9)) for l in range(self.n_levels)]

    def level_sizes(self):
        return [min((r + 1) ** 3, self.table_size) for r in self.resolutions()]

    def dense_flags(self):
        return [(r + 1) ** 3 <= self.table_size for r in self.resolutions()]

    def offsets(self):
        out, o = [], 0
        for sz in self.level_sizes():
            out.append(o)
            o += (sz + 3) // 4 * 4
        return np.array(out + [o], dtype=np.int64)

    @property
    def n_entries(self) -> int:
        return int(self.offsets()[-1])

    @property
    def out_dim(self) -> int:
        return self.n_levels * self.n_feat


def hash_corner_index(spec, level, ix, iy, iz):
    """Entry index (within the level) of integer vertex (ix,iy,iz); uint32 arithmetic."""
    res = spec.resolutions()[level]
    ix = np.asarray(ix).astype(np.uint64).astype(U32)
    iy = np.asarray(iy).astype(np.uint64).astype(U32)
    iz = np.asarray(iz).astype(np.uint64).astype(U32)
    with np.errstate(over="ignore"):
        if spec.dense_flags()[level]:
            s = U32(res + 1)
            return (ix + iy * s + iz * (s * s)).astype(U32)
        h = ix ^ (iy * U32(PRIME_Y)) ^ (iz * U32(PRIME_Z))
        return (h & U32(spec.table_size - 1)).astype(U32)


def hash_cells(spec, x, cmin, cinv):
    """Per level: (i0 (N,3) int64, f (N,3) float32, mask (N,3) bool) -- kernel float32 order."""
    x = np.asarray(x, dtype=F32)
    raw = ((x - np.asarray(cmin, F32)).astype(F32) * np.asarray(cinv, F32)).astype(F32)
    mask = (raw >= F32(0.0)) & (raw <= F32(1.0))
    xn = np.minimum(np.maximum(raw, F32(0.0)), F32(1.0)).astype(F32)
    out = []
    for res in spec.resolutions():
        pos = (xn * F32(res)).astype(F32)
        i0 = np.minimum(np.floor(pos), F32(res - 1)).astype(np.int64)
        f = (pos - i0.astype(F32)).astype(F32)
        out.append((i0, f))
    return out, mask


def hash_encode(spec, x, cmin, cinv, table, dtype=np.float32, return_index=False):
    """x (N,3) canonical points, table (E,F) -> features (N, L*F).

    With ``return_index`` also returns the global entry indices (N, L, 8) uint32 in corner
    order ``(a,b,c)`` = ``a*4 + b*2 + c`` -- the bit-exact parity target.
    """
    dt = np.dtype(dtype).type
    tab = np.asarray(table, dtype=dt)
    cells, _ = hash_cells(spec, x, cmin, cinv)
    offs = spec.offsets()
    n = np.asarray(x).shape[0]
    feats = np.zeros((n, spec.out_dim), dtype=dt)
    idx_all = np.zeros((n, spec.n_levels, 8), dtype=U32)
    for l, (i0, f) in enumerate(cells):
        f = f.astype(dt)
        wx = ((dt(1.0) - f[:, 0]).astype(dt), f[:, 0])
        wy = ((dt(1.0) - f[:, 1]).astype(dt), f[:, 1])
        wz = ((dt(1.0) - f[:, 2]).astype(dt), f[:, 2])
        acc = np.zeros((n, spec.n_feat), dtype=dt)
        for a in (0, 1):
            for b in (0, 1):
                for c in (0, 1):
                    idx = hash_corner_index(spec, l, i0[:, 0] + a, i0[:, 1] + b, i0[:, 2] + c)
                    gidx = idx.astype(np.int64) + offs[l]
                    idx_all[:, l, a * 4 + b * 2 + c] = gidx.astype(U32)
                    wgt = ((wx[a] * wy[b]).astype(dt) * wz[c]).astype(dt)
                    acc = (acc + (wgt[:, None] * tab[gidx]).astype(dt)).astype(dt)
        feats[:, l * spec.n_feat:(l + 1) * spec.n_feat] = acc
    if return_index:
        return feats, idx_all
    return feats


def hash_encode_bwd(spec, x, cmin, cinv, table, dfeat):
    """(d table (E,F) float64, d x (N,3) float64) of ``sum(dfeat * features)``."""
    tab = np.asarray(table, dtype=np.float64)
    cells, mask = hash_cells(spec, x, cmin, cinv)
    offs = spec.offsets()
    res_all = spec.resolutions()
    n = np.asarray(x).shape[0]
    dtab = np.zeros_like(tab)
    dx = np.zeros((n, 3))
    dfeat = np.asarray(dfeat, dtype=np.float64)
    cinv64 = np.asarray(cinv, np.float64)
    for l, (i0, f) in enumerate(cells):
        f = f.astype(np.float64)
        wx = (1.0 - f[:, 0], f[:, 0])
        wy = (1.0 - f[:, 1], f[:, 1])
        wz = (1.0 - f[:, 2], f[:, 2])
        g = dfeat[:, l * spec.n_feat:(l + 1) * spec.n_feat]
        dpos = np.zeros((n, 3))
        for a in (0, 1):
            for b in (0, 1):
                for c in (0, 1):
                    idx = hash_corner_index(spec, l, i0[:, 0] + a, i0[:, 1] + b, i0[:, 2] + c)
                    gidx = idx.astype(np.int64) + offs[l]
                    wgt = wx[a] * wy[b] * wz[c]
                    for ff in range(spec.n_feat):
                        dtab[:, ff] += np.bincount(gidx, weights=wgt * g[:, ff], minlength=tab.shape[0])
                    gv = np.sum(g * tab[gidx], axis=1)
                    sx, sy, sz = (1.0 if a else -1.0), (1.0 if b else -1.0), (1.0 if c else -1.0)
                    dpos[:, 0] += sx * wy[b] * wz[c] * gv
                    dpos[:, 1] += wx[a] * sy * wz[c] * gv
                    dpos[:, 2] += wx[a] * wy[b] * sz * gv
        dx += dpos * res_all[l]
    dx *= cinv64[None, :] * mask
    return dtab, dx
