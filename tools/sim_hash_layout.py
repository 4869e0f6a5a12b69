"""Model of the hash-gather access pattern of k_radiance_tc (lane-paired x-corners, 4
(y, z) corner loads per level per warp) for the current spatial hash vs a 2x2x2
block-interleaved layout: distinct 32-byte sectors / 128-byte lines per warp instruction
and per sample.  Usage: python tools/sim_hash_layout.py"""
import numpy as np
PY, PZ = 2654435761, 805459861
T = 1 << 19
res = [int(np.floor(16 * (2048/16) ** (l/15) + 1e-9)) for l in range(16)]
dense = [(r+1)**3 <= T for r in res]
rng = np.random.default_rng(0)
def idx_cur(l, x, y, z):
    r = res[l]
    if dense[l]:
        s = r + 1
        return x + y*s + z*s*s
    return (x ^ (y*PY & 0xffffffff) ^ (z*PZ & 0xffffffff)) & (T-1)
def idx_blk(l, x, y, z):
    r = res[l]
    sub = (x & 1) | ((y & 1) << 1) | ((z & 1) << 2)
    bx, by, bz = x >> 1, y >> 1, z >> 1
    if dense[l]:
        s = (r + 2) // 2 + 1
        return (bx + by*s + bz*s*s) * 8 + sub
    return (((bx ^ (by*PY & 0xffffffff) ^ (bz*PZ & 0xffffffff)) & (T//8 - 1)) * 8) + sub
def stats(fn, n_warps=400):
    sec = lines = 0; persamp = 0
    for _ in range(n_warps):
        c = rng.uniform(0.1, 0.9, 3); u = rng.normal(size=3); u/=np.linalg.norm(u); v=np.cross(u,[0,0,1.0]); v/=np.linalg.norm(v); w=np.cross(u,v)
        ii, jj = np.meshgrid(np.arange(8), np.arange(4))
        pts = c + 0.0035*(ii.reshape(-1,1)*v + jj.reshape(-1,1)*w)
        for l in range(16):
            p = pts * res[l]
            i0 = np.minimum(np.floor(p).astype(np.int64), res[l]-1)
            for k in range(4):
                b, cc = k >> 1, k & 1
                addrs = []
                for s in range(32):
                    for a in range(2):
                        addrs.append(fn(l, i0[s,0]+a, i0[s,1]+b, i0[s,2]+cc) * 4)
                addrs = np.array(addrs)
                sec += len(np.unique(addrs // 32)); lines += len(np.unique(addrs // 128))
            for s in range(32):
                a8 = [fn(l, i0[s,0]+a, i0[s,1]+b, i0[s,2]+cc)*4 for a in range(2) for b in range(2) for cc in range(2)]
                persamp += len(set(x//32 for x in a8))
    n = n_warps*16
    return sec/n, lines/n, persamp/(n*32)
print("current: sectors/level-warp-instr-quad %.1f lines %.1f  sectors per sample-level %.2f" % stats(idx_cur))
print("block  : sectors/level-warp-instr-quad %.1f lines %.1f  sectors per sample-level %.2f" % stats(idx_blk))
