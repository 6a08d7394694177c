"""Summarise ncu reports (--page raw) into a small markdown table for profiles/.

usage: python tools/ncu_summary.py out.md rep1.ncu-rep [rep2 ...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st conflicts"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long-sb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for line in r[2:]:
        d = dict(zip(hdr, line))
        u = dict(zip(hdr, units))
        yield d, u


def main():
    out, reps = sys.argv[1], sys.argv[2:]
    lines = ["| report | kernel | grid | " + " | ".join(k[1] for k in KEYS) + " |",
             "|---" * (3 + len(KEYS)) + "|"]
    for rep in reps:
        for d, u in rows(rep):
            vals = [f"{d.get(k, '')} {u.get(k, '')}".strip() for k, _ in KEYS]
            name = d.get("Kernel Name", "")[:48]
            lines.append(f"| {rep.split('/')[-1]} | `{name}` | {d.get('Grid Size', '')} | " + " | ".join(vals) + " |")
    with open(out, "a") as fh:
        fh.write("\n".join(lines) + "\n\n")


if __name__ == "__main__":
    main()
