"""Aggregate warp-stall samples of one kernel by reason, and by SASS opcode class.

    python scripts/ncu_stalls.py gpurun_out/x_full.ncu-rep <kernel-regex>
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main(rep, kre):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ci = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    seen, body = set(), []
    for r in rows[2:]:
        if len(r) != len(hdr) or r[0] in seen:
            continue
        seen.add(r[0])
        body.append(r)

    def num(x):
        try:
            return int(x.replace(",", ""))
        except ValueError:
            return 0
    by_reason = collections.Counter()
    by_op = collections.Counter()
    for r in body:
        op = r[ci["Source"]].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", op).split(" ")[0].split(".")[0]
        tot = num(r[ci["Warp Stall Sampling (All Samples)"]])
        by_op[op] += tot
        for c in stall_cols:
            by_reason[c[6:]] += num(r[ci[c]])
    T = sum(by_reason.values())
    print("by reason:")
    for k, v in by_reason.most_common(14):
        print(f"  {k:24s} {v:9d} {100 * v / T:5.1f}%")
    T2 = sum(by_op.values())
    print("by opcode:")
    for k, v in by_op.most_common(24):
        print(f"  {k:24s} {v:9d} {100 * v / T2:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
