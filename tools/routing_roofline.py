"""Summarise an ncu CSV of the routing / gate kernels of one step (dev tool, not product).

    python tools/routing_roofline.py CSV CONFIG R_PAD R_MEAN OUT.json [--peak 6556.2]

CSV: `ncu -i REP --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum,...` of a `bench.py --no-graph --steps 1 --warmup 1` capture; the LAST
occurrence of every kernel (the timed step) is kept.  Each kernel's ALGORITHMIC bytes (what the
operation must move at least once: SURVEY §8(d) terms, GEMM operand traffic excluded) are set
against its time (achieved GB/s, fraction of the HBM peak) and against ncu's DRAM bytes (traffic
ratio: > 1 means re-reads; < 1 means L2 served part of it -- ncu flushes caches before each
replay, but small outputs can stay in L2 when the kernel ends).
"""
import csv
import json
import re
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from harness import configs  # noqa: E402

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def algorithmic_bytes(cfg, R, Rp):
    """name pattern -> (bytes, what) per launch at this config (b = bytes per activation)."""
    b = 2 if cfg.dtype == "bf16" else 4
    T, d, f, E = cfg.T, cfg.d_model, cfg.d_ff, cfg.E
    Ep = (E + 15) // 16 * 16
    Kp = (2 * Ep + 63) // 64 * 64
    words = (d * f + 31) // 32
    return [
        (r"spawn_kernel", d * f * b + E * words * 4 + E * d * f * b, "read W_s + E mask words, write E masked copies"),
        (r"gate_fused_tc_kernel", T * d * b + T * E * 4 * 3, "read x, u; write probs, slot"),
        (r"gate_fused_kernel", T * d * b + T * E * 4 * 3, "read x, u; write probs, slot"),
        (r"dispatch_rank_kernel", T * E * 4 * 3 + Rp * 8, "read probs, slot; write slot, row_token, row_gate"),
        (r"dispatch_copy_kernel", T * d * b + Rp * d * b, "read x once, write x_perm (pads zero)"),
        (r"combine_bwd_colsum_kernel", T * d * b + R * d * b + Rp * d * b + Rp * 12,
         "read dy (each token once) + e_out, write d_eout (+ dG, meta)"),
        (r"combine_kernel", R * d * b + T * d * b + T * E * 4 + R * 4, "read e_out rows + slot + gates, write y"),
        (r"gate_bwd_token_kernel|gate_bwd_quad_kernel", 3 * T * E * 4 + R * 4 + T * Kp * 2, "read probs, slot, dG; write dlogits + bf16 hi|lo"),
        (r"gate_tc_kernel<2>", T * d * b + T * Kp * 2, "dW_g: read x, dL hi|lo"),
        (r"tc_gemm_kernel<3, false, false, false, 0>|tc_gemm_kernel<3, 0, 0, 0", T * Kp * 2 + T * d * b,
         "dL W_g^T: read dL hi|lo, write dx"),
        (r"dispatch_bwd_kernel", T * E * 4 + R * d * b + 2 * T * d * b, "read slot, dx_perm rows, dx; write dx"),
        (r"colsum_part_kernel", Rp * f * 4 // 32, "db1 partials (fp32 [R/32, f]) read"),
    ]


def main():
    path, name, Rp, R, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(float(sys.argv[4])), sys.argv[5]
    peak = float(sys.argv[sys.argv.index("--peak") + 1]) if "--peak" in sys.argv else 6556.2
    cfg = configs.get(name)
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, units = rows[hi], rows[hi + 1]
    col = {h: i for i, h in enumerate(hdr)}
    last = {}
    for r in rows[hi + 2:]:
        k = r[col["Kernel Name"]]
        key = re.sub(r"\(.*", "", k)
        last[key] = r                       # keep the last launch of each kernel (the timed step)
    formulas = algorithmic_bytes(cfg, R, Rp)
    table = []
    for key, r in last.items():
        us = float(r[col["gpu__time_duration.sum"]]) * SCALE[units[col["gpu__time_duration.sum"]]]
        rd = float(r[col["dram__bytes_read.sum"]]) * SCALE[units[col["dram__bytes_read.sum"]]]
        wr = float(r[col["dram__bytes_write.sum"]]) * SCALE[units[col["dram__bytes_write.sum"]]]
        alg, what = None, None
        for pat, byts, w in formulas:
            if re.search(pat, key):
                alg, what = byts, w
                break
        row = {"kernel": key.replace("void ", "").replace("unnamed>::", ""), "us": us, "dram_bytes": rd + wr}
        if alg:
            row.update(algorithmic_bytes=alg, what=what, achieved_gbs=alg / us * 1e-3,
                       frac_of_hbm_peak=alg / us * 1e-3 / peak, traffic_ratio=(rd + wr) / alg)
        table.append(row)
    json.dump({"workload": name, "rows_R_pad": Rp, "rows_R": R, "hbm_peak_gbs": peak, "source": path,
               "kernels": table}, open(out, "w"), indent=1)
    for t in table:
        if "algorithmic_bytes" in t:
            print(f'{t["kernel"][:48]:48s} {t["us"]:8.1f} us  alg {t["algorithmic_bytes"]/1e6:8.1f} MB  '
                  f'{t["achieved_gbs"]:7.0f} GB/s ({t["frac_of_hbm_peak"]:.2f})  traffic x{t["traffic_ratio"]:.2f}')
        else:
            print(f'{t["kernel"][:48]:48s} {t["us"]:8.1f} us  (latency-bound helper, {t["dram_bytes"]/1e6:.2f} MB)')


if __name__ == "__main__":
    main()
