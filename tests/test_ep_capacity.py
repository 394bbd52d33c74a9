"""The peer-memory EP path's row-capacity rule (paper_2112_14397_b200.ep2.EP2Rank), host side.

VERDICT r1 missing #2: the static worst case R_cap = W*T*E_local (every rank's tokens to every
local expert) is 8.4 M rows per rank at C4 -- ~206 GB of [R_cap, d_ff] / [R_cap, d] row buffers,
more than a B200 holds.  The capacity is now sized from the all-gathered counts ("adaptive
capacity"): the largest rank's 128-aligned recv layout times a headroom factor.  CPU only.
"""
import numpy as np

from harness import configs, inputs
from oracle import dts_moe as O


def _rank(W, cfg, headroom=1.25):
    from paper_2112_14397_b200.ep2 import EP2Rank
    r = EP2Rank.__new__(EP2Rank)          # the sizing rule only: no context, no device
    r.world, r.El, r.T, r.E, r.headroom = W, cfg.E // W, cfg.T, cfg.E, headroom
    return r


def test_rows_needed_is_the_largest_recv_layout():
    cfg = configs.C3
    r = _rank(4, cfg)
    ca = np.zeros((4, cfg.E), np.int64)
    ca[0, 0] = 1            # expert 0 (rank 0): 1 row -> 128
    ca[1, 9] = 300          # expert 9 (rank 1): 300 rows + 300 from rank 2 -> 640
    ca[2, 9] = 300
    ca[3, 31] = 129         # expert 31 (rank 3): 256
    assert r.rows_needed(ca) == 640
    assert r.capacity_for(ca) == 896          # ceil(640 * 1.25) = 800 -> 128-aligned 896
    assert r.round_rows(0) == 128


def test_c4_capacity_fits_hbm():
    cfg = configs.C4
    li = inputs.make_inputs(cfg, T=16384)
    p = O.gumbel_softmax(inputs.to_f64(li.x), inputs.to_f64(li.Wg), inputs.to_f64(li.u), float(np.float32(cfg.tau)))
    m = O.threshold_select(p, float(np.float32(cfg.threshold)))
    counts = m.sum(0).astype(np.int64) * (cfg.T // 16384)          # one rank's full-T counts
    row_bytes = (2 * cfg.d_ff + 4 * cfg.d_model) * 2                 # gp, h + x_recv, e_out, d_eout, dx_perm
    for W in (1, 2, 4, 8):
        r = _rank(W, cfg)
        cap = r.capacity_for(np.tile(counts, (W, 1)))                # W ranks with this load (weak scaling)
        gb, worst = cap * row_bytes / 1e9, r.worst_case_capacity() * row_bytes / 1e9
        print(f"C4 W={W}: {cap} rows -> {gb:.1f} GB of row buffers (worst case {worst:.0f} GB)")
        assert gb < 10 and worst > 180
