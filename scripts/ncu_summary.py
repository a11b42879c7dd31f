"""Summarise an ncu --set full report of the PSN stream kernels into a small
markdown table (committed under profiles/) and a JSON of per-launch DRAM
traffic that bench.py reports as roofline.traffic.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_ncu_stream.md profiles/ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration (us)", 1e-3),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1.0),
    ("dram__bytes_write.sum", "DRAM write (MB)", 1.0),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)", 1.0),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate (%)", 1.0),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe (% of peak)", 1.0),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe (% of peak)", 1.0),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)", 1.0),
    ("launch__registers_per_thread", "registers / thread", 1.0),
    ("launch__grid_size", "grid (CTAs)", 1.0),
    ("launch__block_size", "block (threads)", 1.0),
]


def main(rep, md_out, json_out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    lines = ["| kernel | " + " | ".join(m[1] for m in METRICS) + " | stall mix |", "|---" * (len(METRICS) + 2) + "|"]
    traffic = {}
    for r in data:
        name = r[col["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")
        if "psn_stream_kernel" in short:
            tmpl = name[name.index("<") + 1:name.index(">")]
            short = "psn_stream_kernel<" + tmpl + ">"
        vals = []
        for key, _, scale in METRICS:
            v = r[col[key]] if key in col else ""
            try:
                f = float(v.replace(",", ""))
                unit = units[col[key]] if key in col else ""
                if key.startswith("dram__bytes"):
                    f = f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
                elif key == "gpu__time_duration.sum":
                    f = f * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1.0)
                vals.append(f"{f:.1f}")
            except ValueError:
                vals.append(v)
        stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i] or 0)) for h, i in col.items()
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        tot = sum(v for _, v in stalls) or 1.0
        mix = ", ".join(f"{h} {100 * v / tot:.0f}%" for h, v in sorted(stalls, key=lambda t: -t[1])[:4])
        lines.append(f"| {short} | " + " | ".join(vals) + f" | {mix} |")
        try:
            rd = float(vals[1]) * 1e6
            wr = float(vals[2]) * 1e6
            traffic[short] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr,
                              "duration_us_under_ncu": float(vals[0])}
        except ValueError:
            pass
    with open(md_out, "w") as f:
        f.write(f"ncu --set full summary of `{rep}` (per launch; times are ncu-serialised, cold-cache)\n\n")
        f.write("\n".join(lines) + "\n")
    with open(json_out, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
