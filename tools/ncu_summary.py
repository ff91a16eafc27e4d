"""Summarise an ncu --set full report (.ncu-rep) into the metrics DESIGN.md cites (one row per kernel).

usage: python tools/ncu_summary.py REPORT.ncu-rep [OUT.md] [--traffic-key CONFIG:kK]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("time_ms", "gpu__time_duration.sum", 1e-6),
    ("dram_read_GB", "dram__bytes_read.sum", 1e-9),
    ("dram_write_GB", "dram__bytes_write.sum", 1e-9),
    ("l1tex_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    ("lts_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("inst_G", "smsp__inst_executed.sum", 1e-9),
    ("smem_wavefronts_M", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1e-6),
    ("smem_bank_conflicts_M", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1e-6),
    ("gld_sectors_M", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 1e-6),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct", 1),
]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "msecond": 1e6, "usecond": 1e3, "nsecond": 1,
        "ms": 1e6, "us": 1e3, "ns": 1}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        r = {"kernel": d[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for name, m, scale in METRICS:
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(d[i].replace(",", ""))
            except ValueError:
                continue
            v *= UNIT.get(units[i], 1)
            r[name] = v * scale
        res.append(r)
    return res


def main():
    rep = sys.argv[1]
    res = load(rep)
    cols = ["kernel"] + [n for n, _, _ in METRICS]
    lines = ["| " + " | ".join(cols) + " |", "|" + "---|" * len(cols)]
    for r in res:
        lines.append("| " + " | ".join(f"{r.get(c, ''):.4g}" if isinstance(r.get(c), float) else str(r.get(c, ""))
                                       for c in cols) + " |")
    text = "\n".join(lines)
    if len(sys.argv) > 2 and not sys.argv[2].startswith("--"):
        with open(sys.argv[2], "w") as f:
            f.write(f"ncu --set full summary of {rep}\n\n" + text + "\n")
    print(text)
    if "--traffic-key" in sys.argv:
        key = sys.argv[sys.argv.index("--traffic-key") + 1]
        print(json.dumps({f"{key}:{r['kernel'].split('<')[0].split('::')[-1]}": (r['dram_read_GB'] + r['dram_write_GB']) * 1e9
                          for r in res}))


if __name__ == "__main__":
    main()
