"""Summarise ncu reports into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py gpurun_out/prof_k3.ncu-rep [more.ncu-rep] > profiles/x.md
Writes/updates profiles/ncu_summary.json with dram bytes per launch per kernel
(bench.py reads it for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "smsp__cycles_active.avg"]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "byte": 1.0,
         "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        res.append(d)
    return res


def top_stalls(rep, k=8):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    col = idx.get("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((float(r[col] or 0), r[1]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1.0
    return [(100 * s / tot, src) for s, src in sorted(data, reverse=True)[:k]]


def main():
    summ_path = os.path.join("profiles", "ncu_summary.json")
    try:
        summary = json.load(open(summ_path))
    except (OSError, ValueError):
        summary = {}
    for rep in sys.argv[1:]:
        for d in raw(rep):
            name = d.get("Kernel Name", ("?", ""))[0]
            short = name.split("(")[0].split()[-1].split("::")[-1].split("<")[0]
            print(f"## {short}  ({os.path.basename(rep)})\n")
            print(f"`{name}`\n")
            for key in KEYS:
                if key in d:
                    v, u = d[key]
                    print(f"- {key}: {v} {u}")
            rd = float(d["dram__bytes_read.sum"][0]) * SCALE.get(d["dram__bytes_read.sum"][1], 1)
            wr = float(d["dram__bytes_write.sum"][0]) * SCALE.get(d["dram__bytes_write.sum"][1], 1)
            t = float(d["gpu__time_duration.sum"][0]) * SCALE.get(d["gpu__time_duration.sum"][1], 1)
            print(f"- dram bytes per launch (read+write): {rd + wr:.4e}  over {t * 1e3:.3f} ms "
                  f"= {(rd + wr) / t / 1e9:.0f} GB/s\n")
            print("Top warp-stall sites (share of samples, SASS):\n")
            for pct, src in top_stalls(rep):
                print(f"- {pct:5.1f}%  `{src.strip()[:90]}`")
            print()
            summary[short] = {"dram_bytes_per_launch": rd + wr, "duration_s_under_ncu": t,
                              "tensor_active_pct": d.get(KEYS[3], ("", ""))[0],
                              "report": os.path.basename(rep)}
    with open(summ_path, "w") as fh:
        json.dump(summary, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
