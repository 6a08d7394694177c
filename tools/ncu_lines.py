"""Per-source-line warp-stall samples and executed instructions of one kernel
in an ncu report (--import-source on, -lineinfo build):

  python tools/ncu_lines.py report.ncu-rep 'k_fft8<(int)4' [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, key = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fn = path = hdr = None
    samp, inst = collections.Counter(), collections.Counter()
    why = collections.defaultdict(collections.Counter)
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
        elif r[0] == "Function Name":
            fn = r[1]
        elif r[0] == "Line No":
            hdr = r
        elif fn and key in fn and hdr and len(r) > 8 and r[0].isdigit():
            k = (path, int(r[0]), r[1][:80].strip())
            try:
                samp[k] += int(r[hdr.index("Warp Stall Sampling (All Samples)")])
                inst[k] += int(r[hdr.index("Instructions Executed")])
                for c, name in enumerate(hdr):
                    if name.startswith("stall_") and "Not Issued" not in name and r[c] not in ("", "0"):
                        why[k][name[6:]] += int(r[c])
            except ValueError:
                pass
    ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
    print(f"samples {ts}  warp instructions {ti}")
    for k, v in samp.most_common(top):
        w = " ".join(f"{n}:{c}" for n, c in why[k].most_common(3))
        print(f"{v:6d} {100 * v / ts:5.1f}%  inst {100 * inst[k] / ti:5.1f}%  {k[0]}:{k[1]} {k[2][:60]}  [{w}]")


if __name__ == "__main__":
    main()
