"""Per-launch hardware counters of one kernel from an ncu report, merged into profiles/ncu_counters.json (tracked):
the numbers bench.py's `roofline` block divides by its LIVE launch time (the Table 2
ncu method of PAPER.md:541-555).

usage: python tools/ncu_counters.py REPORT.ncu-rep KEY [--source TEXT]      KEY = config:kK:kernel (e.g. reddit:k32:fwd)

Counters (per launch): dram_bytes (read + write), l1tex_wavefronts (all LSU data-pipe wavefronts = SM average x
SM count), smem_wavefronts, smem_bank_conflicts, inst (warp instructions), lts_red_sectors / lts_atom_sectors
(when the capture added them with --metrics), time_ms and sm_ghz under the profiler (for reference only).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.environ.get("NCU_COUNTERS_OUT", os.path.join(ROOT, "profiles", "ncu_counters.json"))
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9,
        "Ghz": 1e9, "Mhz": 1e6, "hz": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "GHz": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, key = sys.argv[1], sys.argv[2]
    src = sys.argv[sys.argv.index("--source") + 1] if "--source" in sys.argv else os.path.basename(rep)
    hdr, units, data = raw(rep)
    d = data[-1]

    def get(name):
        if name not in hdr:
            return None
        i = hdr.index(name)
        try:
            v = float(d[i].replace(",", ""))
        except ValueError:
            return None
        return v * UNIT.get(units[i], 1)

    n_sm = get("device__attribute_multiprocessor_count") or 148
    lsu_avg = get("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg")
    rec = {
        "kernel": d[hdr.index("Kernel Name")].split("(")[0].replace("void ", ""),
        "time_ms_under_ncu": (get("gpu__time_duration.sum") or 0) * 1e3,
        "sm_ghz_under_ncu": (get("sm__cycles_elapsed.avg.per_second") or 0) / 1e9,
        "dram_bytes": (get("dram__bytes_read.sum") or 0) + (get("dram__bytes_write.sum") or 0),
        "l1tex_wavefronts": lsu_avg * n_sm if lsu_avg is not None else get("l1tex__data_pipe_lsu_wavefronts.sum"),
        "l1tex_pct_of_peak_under_ncu": get("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed"),
        "smem_wavefronts": get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "smem_bank_conflicts": get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "inst": get("smsp__inst_executed.sum"),
        "issue_active_pct_under_ncu": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "lts_red_sectors": get("lts__t_sectors_op_red.sum"),
        "lts_atom_sectors": get("lts__t_sectors_op_atom.sum"),
        "l2_hit_pct": get("lts__t_sector_hit_rate.pct"),
        "n_sm": n_sm,
        "source": src,
    }
    allc = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            allc = json.load(f)
    allc[key] = rec
    with open(OUT, "w") as f:
        json.dump(allc, f, indent=1, sort_keys=True)
    print(json.dumps({key: rec}))


if __name__ == "__main__":
    main()
