"""Summarise an ncu SASS source page (ncu -i X --page source --csv --print-source sass):
instruction mix weighted by executions, and stall samples by opcode."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {k: i for i, k in enumerate(hdr)}
    by_op = collections.Counter()
    stall = collections.Counter()
    total = 0
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        try:
            n = int(r[ix["Instructions Executed"]] or 0)
            s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        by_op[op] += n
        stall[op] += s
        total += n
    print(f"total warp instructions executed: {total:,}")
    tot_s = sum(stall.values())
    for op, n in by_op.most_common(top):
        print(f"{op:28s} {n:16,d} {100.0 * n / total:6.2f}%   stall-samples {100.0 * stall[op] / max(tot_s, 1):6.2f}%")


if __name__ == "__main__":
    main(sys.argv[1])
