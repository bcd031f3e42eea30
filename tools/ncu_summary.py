"""Summarise an ncu report: time, pipes, issue, occupancy, DRAM, top stalls.
usage: python tools/ncu_summary.py report.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "time_ms": ("gpu__time_duration.sum", 1.0),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "fma_inst_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    "alu_pipe_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "xu_inst_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    "lsu_inst_pct": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "regs": ("launch__registers_per_thread", 1),
    "warp_inst": ("smsp__inst_executed.sum", 1),
    "threads_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    "dram_read_MB": ("dram__bytes_read.sum", 1),
    "dram_write_MB": ("dram__bytes_write.sum", 1),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
    "sm_clock_ghz": ("smsp__cycles_elapsed.avg.per_second", 1),
}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k, (m, _) in KEYS.items():
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                u = units[hdr.index(m)]
                try:
                    x = float(v)
                except ValueError:
                    continue
                if u == "Mbyte" or u == "MB":
                    pass
                elif u in ("Kbyte", "KB"):
                    x /= 1e3
                elif u in ("byte",):
                    x /= 1e6
                elif u in ("Gbyte", "GB"):
                    x *= 1e3
                if k == "time_ms":
                    x = {"nsecond": x / 1e6, "ns": x / 1e6, "usecond": x / 1e3, "us": x / 1e3, "msecond": x, "ms": x, "second": x * 1e3, "s": x * 1e3}.get(u, x)
                d[k] = x
        stalls = []
        for k, v in zip(hdr, r):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", ""))))
                except ValueError:
                    pass
        tot = sum(v for _, v in stalls) or 1.0
        d["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls, key=lambda x: -x[1])[:8]}
        res.append(d)
    return res


if __name__ == "__main__":
    res = load(sys.argv[1])
    for d in res:
        print(json.dumps(d))
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
