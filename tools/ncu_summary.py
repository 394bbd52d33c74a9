"""Summarise an `ncu --set full` report of the expert GEMM kernels into a JSON that bench.py
reads for roofline.traffic (dram bytes per step of the GEMM set).  Dev tool, not product.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep WORKLOAD profiles/r01/ncu_gemm_WORKLOAD.json
"""
import csv
import io
import json
import re
import subprocess
import sys

MET = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size"]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "%": 1.0, "": 1.0}
ROLE = {"<0, 0, 0, 0>": "GEMM1 a=x W1+b1 -> h,gp", "<1, 0, 0, 0>": "GEMM2 o=h W2+b2",
        "<2, 0, 1, 0>": "dgrad2 da=(do W2^T)*gp (+db1)", "<3, 0, 1, 0>": "dgrad1 dx=da W1^T",
        "<4, 1, 1, 1>": "wgrad (dW1 or dW2, KGRP)", "<3, 0, 0, 0>": "gate dL W_g^T (dense)"}


def main():
    rep, workload, out = sys.argv[1], sys.argv[2], sys.argv[3]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(MET)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    kern = []
    for r in rows[2:]:
        d = {}
        for m in MET:
            i = hdr.index(m)
            d[m] = float(r[i]) * SCALE.get(units[i], 1.0)
        name = r[hdr.index("Kernel Name")]
        mt = re.search(r"tc_gemm_kernel(<[^>]*>)", name)
        tmpl = mt.group(1) if mt else name
        kern.append({"kernel": "tc_gemm_kernel" + tmpl, "role": ROLE.get(tmpl, ROLE.get(re.sub(r", \d+>$", ">", tmpl), "?")),   # 5th parameter: epilogue warp override
                     "us": d[MET[0]], "dram_read_bytes": d[MET[1]], "dram_write_bytes": d[MET[2]],
                     "tensor_pipe_pct": d[MET[3]], "sm_throughput_pct": d[MET[4]]})
    experts = [k for k in kern if not k["role"].startswith("gate")]
    summ = {"workload": workload, "report": rep.split("/")[-1], "kernels": kern,
            "expert_gemm_set": {"launches": len(experts), "us": sum(k["us"] for k in experts),
                                "dram_bytes": sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in experts)}}
    json.dump(summ, open(out, "w"), indent=1)
    for k in kern:
        print(f'{k["role"][:34]:34s} {k["us"]:8.1f} us  rd {k["dram_read_bytes"]/1e9:6.3f} GB  wr {k["dram_write_bytes"]/1e9:6.3f} GB  tensor {k["tensor_pipe_pct"]:5.1f}%')
    print(summ["expert_gemm_set"])


if __name__ == "__main__":
    main()
