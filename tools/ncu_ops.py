"""Executed warp instructions by SASS opcode for one kernel of an ncu report.
usage: python tools/ncu_ops.py REPORT KERNEL_REGEX UNITS [TOP]"""
import csv
import subprocess
import sys


def main(rep, kern, units, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    ops = {}
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        try:
            ie = int(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        src = r[hdr.index("Source")].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        ops[op] = ops.get(op, 0) + ie
    tot = sum(ops.values()) or 1
    print(f"total warp instructions per unit {tot / float(units):.0f}")
    for op, v in sorted(ops.items(), key=lambda x: -x[1])[:int(top)]:
        print(f"  {op:24s} {v / float(units):10.0f} {v / tot:6.3f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
