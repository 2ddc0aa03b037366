"""Instruction mix of one kernel from an ncu report's SASS source page.

    python tools/sass_mix.py <report.ncu-rep> <launch-skip> [warps]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, skip = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    print(rows[0][1][:100])
    hdr = rows[1]
    ix, src = hdr.index("Instructions Executed"), hdr.index("Source")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    ops, stalls = collections.Counter(), collections.Counter()
    tot = 0
    for r in rows[2:]:
        if len(r) < len(hdr) or not r[ix].strip().isdigit():
            continue
        n = int(r[ix])
        tot += n
        toks = r[src].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        ops[op.split(".")[0]] += n
        stalls[op.split(".")[0]] += int(r[st] or 0)
    warps = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    print(f"total warp instructions {tot}  per warp {tot / warps:.1f}")
    for k, v in ops.most_common(30):
        print(f"  {k:10s} {v / warps:8.1f}   stall samples {stalls[k]}")


if __name__ == "__main__":
    main()
