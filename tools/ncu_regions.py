"""Executed warp instructions per unit, bucketed by (file, line range) regions of one kernel.
usage: python tools/ncu_regions.py REPORT KERNEL_REGEX UNITS FILE:START-END=name ..."""
import collections
import csv
import subprocess
import sys


def main(rep, kern, units, *specs):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, fname, res = None, None, collections.Counter()
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "":
            continue
        try:
            res[(fname, int(r[0]))] += int(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            pass
    regs = []
    for sp in specs:
        loc, name = sp.split("=")
        f, rng = loc.split(":")
        a, b = rng.split("-")
        regs.append((f, int(a), int(b), name))
    b = collections.Counter()
    for (f, l), v in res.items():
        nm = next((n for ff, a, bb, n in regs if ff == f and a <= l <= bb), f)
        b[nm] += v
    tot = sum(b.values()) or 1
    print(f"total per unit {tot / float(units):.0f}")
    for k, v in b.most_common():
        print(f"  {k:28s} {v / float(units):9.0f} {v / tot:.3f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
