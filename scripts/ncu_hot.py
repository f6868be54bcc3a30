"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.

    python scripts/ncu_hot.py gpurun_out/x_full.ncu-rep <kernel-regex> [N]
"""
import csv
import io
import subprocess
import sys


def main(rep, kre, n=40):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ci = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_")]
    def num(x):
        try:
            return int(x.replace(",", ""))
        except ValueError:
            return None
    body = [r for r in rows[2:] if len(r) == len(hdr) and num(r[ci["Warp Stall Sampling (All Samples)"]]) is not None]
    tot = sum(num(r[ci["Warp Stall Sampling (All Samples)"]]) for r in body)
    print(f"total samples {tot}, instructions {len(body)}")
    body.sort(key=lambda r: -num(r[ci["Warp Stall Sampling (All Samples)"]]))
    for r in body[:n]:
        s = num(r[ci["Warp Stall Sampling (All Samples)"]])
        st = sorted((((num(r[ci[c]]) or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        sts = " ".join(f"{c}:{v}" for v, c in st if v)
        print(f"{s:6d} {100.0 * s / max(tot, 1):5.1f}% {r[ci['Address']][-5:]} {r[ci['Source']].strip()[:60]:60s} {sts}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
