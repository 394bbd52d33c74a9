"""Analyse a MOE_EXP_TRACE dump (gpurun_out/trace_<EPI>.bin): per-warp event log of CTAs 0, 1."""
import sys
import numpy as np
N = 4096
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(2, 16, N)
names = {1: 'prod_empty_wait0', 2: 'prod_empty_wait1', 3: 'mma_tempty0', 4: 'mma_tempty1', 5: 'mma_full1',
         6: 'epi_tfull0', 7: 'epi_tfull1', 8: 'epi_ldwait', 9: 'epi_commit', 10: 'epi_tile_end', 11: 'epi_math_end',
         12: 'epi_fence_end'}
for cta in range(2):
    for w in range(16):
        ev = a[cta, w]
        ev = ev[ev != 0]
        if len(ev) == 0:
            continue
        typ = (ev >> 56).astype(int); tile = ((ev >> 40) & 0xffff).astype(int); clk = (ev & 0xFFFFFFFFFF).astype(np.int64)
        clk = clk - clk[0]
        if w == int(sys.argv[2]) if len(sys.argv) > 2 else False:
            for i in range(min(len(ev), 120)):
                print(cta, w, names.get(typ[i], typ[i]), tile[i], clk[i])
        # summary
        span = clk[-1]
        if w >= 2:
            # time waiting for tfull
            wt = 0; tiles = 0; math = 0; ld = 0; fence = 0; store = 0
            last6 = None; lastc = None
            for i in range(len(ev)):
                if typ[i] == 6: last6 = clk[i]
                if typ[i] == 7 and last6 is not None: wt += clk[i] - last6; tiles += 1; lastc = clk[i]
                if typ[i] == 8 and lastc is not None: ld += clk[i] - lastc; lastc = clk[i]
                if typ[i] == 11 and lastc is not None: math += clk[i] - lastc; lastc = clk[i]
                if typ[i] == 12 and lastc is not None: fence += clk[i] - lastc; lastc = clk[i]
                if typ[i] == 9 and lastc is not None: store += clk[i] - lastc; lastc = clk[i]
            print(f"cta{cta} w{w:2d} span {span:8d} tiles {tiles:3d} per-tile {span/max(tiles,1):7.0f}  tfull-wait {wt/max(tiles,1):6.0f} "
                  f"ld+wait {ld/max(tiles,1):6.0f} math {math/max(tiles,1):6.0f} fence {fence/max(tiles,1):5.0f} store {store/max(tiles,1):5.0f}")
        elif w == 1 and cta == 0:
            wt = 0; n = 0; l3 = None
            for i in range(len(ev)):
                if typ[i] == 3: l3 = clk[i]
                if typ[i] == 4 and l3 is not None: wt += clk[i] - l3; n += 1
            print(f"cta{cta} MMA span {span} tiles {n} tempty-wait/tile {wt/max(n,1):.0f}")

# MMA warp: gaps between consecutive k-block 'full acquired' events, and producer empty waits
ev = a[0, 1]; ev = ev[ev != 0]
typ = (ev >> 56).astype(int); clk = (ev & 0xFFFFFFFFFF).astype(np.int64)
t5 = clk[typ == 5]
g = np.diff(t5)
print("MMA k-block gaps: n", len(g), "mean", g.mean(), "p50", np.median(g), "p90", np.percentile(g, 90), "max", g.max())
for cta in range(2):
    ev = a[cta, 0]; ev = ev[ev != 0]
    typ = (ev >> 56).astype(int); clk = (ev & 0xFFFFFFFFFF).astype(np.int64)
    w = clk[1:][(typ[1:] == 2) & (typ[:-1] == 1)] - clk[:-1][(typ[1:] == 2) & (typ[:-1] == 1)]
    i2 = clk[typ == 2]
    print(f"producer cta{cta}: empty-wait mean {w.mean():.0f}  issue interval mean {np.diff(i2).mean():.0f}")
