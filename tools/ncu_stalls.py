"""Summarise warp-stall samples of an ncu report by reason and by hot SASS line.

Development tool:  python tools/ncu_stalls.py REPORT.ncu-rep [--kernel REGEX] [--min-exec N] [--top K]
(`ncu -i REPORT --page source --csv --print-source sass` underneath).
--min-exec/--max-exec restrict to instructions executed that many times (e.g. one loop body).
"""

import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--min-exec", type=int, default=0)
    ap.add_argument("--max-exec", type=int, default=1 << 62)
    ap.add_argument("--top", type=int, default=25)
    args = ap.parse_args()
    cmd = ["ncu", "-i", args.report, "--page", "source", "--csv", "--print-source", "sass"]
    if args.kernel:
        cmd += ["-k", f"regex:{args.kernel}"]
    txt = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr, data = rows[hi], [r for r in rows[hi + 1:] if len(r) == len(rows[hi])]
    col = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]

    def num(r, h):
        v = r[col[h]].replace(",", "")
        return int(v) if v.isdigit() else 0

    sel = [r for r in data if args.min_exec <= num(r, "Instructions Executed") <= args.max_exec]
    tot = collections.Counter()
    for r in sel:
        for h in reasons:
            tot[h] += num(r, h)
    insts = sum(num(r, "Instructions Executed") for r in sel)
    samples = sum(num(r, "Warp Stall Sampling (All Samples)") for r in sel)
    print(f"{len(sel)} SASS lines, {insts} warp-instructions executed, {samples} samples")
    for h, v in tot.most_common():
        if v:
            print(f"  {h:28s} {v:7d} {100 * v / max(samples, 1):5.1f}%")
    print("hot lines:")
    for r in sorted(sel, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[: args.top]:
        top = max(reasons, key=lambda h: num(r, h))
        print(f"  {num(r, 'Warp Stall Sampling (All Samples)'):5d} exec={num(r, 'Instructions Executed'):7d} "
              f"{top[6:]:14s} {r[col['Source']].strip()[:80]}")


if __name__ == "__main__":
    main()
