"""Executed warp instructions AND stall samples per unit, bucketed by source-line regions of one
kernel (every file's source rows, inline-asm lines included).
usage: python tools/ncu_regions2.py REPORT KERNEL_REGEX UNITS FILE:START-END=name ..."""
import collections
import subprocess
import sys


def main(rep, kern, units, *specs):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    ins, smp = collections.Counter(), collections.Counter()
    fname, hdr = None, None
    for line in out.splitlines():
        # ncu does not escape quotes inside the source column: split on the field separator
        r = line.strip().strip('"').split('","') if line.strip() else []
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        k = (fname, int(r[0]))
        num = lambda x: int(x) if x.isdigit() else 0
        ins[k] += num(r[hdr.index("Instructions Executed")])
        smp[k] += num(r[hdr.index("Warp Stall Sampling (All Samples)")])
    regs = []
    for sp in specs:
        loc, name = sp.split("=")
        f, rng = loc.split(":")
        a, b = rng.split("-")
        regs.append((f, int(a), int(b), name))
    bi, bs = collections.Counter(), collections.Counter()
    for (f, l), v in ins.items():
        nm = next((n for ff, a, bb, n in regs if ff == f and a <= l <= bb), f)
        bi[nm] += v
        bs[nm] += smp[(f, l)]
    ti, ts = sum(bi.values()) or 1, sum(bs.values()) or 1
    print(f"total warp instructions per unit {ti / float(units):.0f}")
    print(f"  {'region':28s} {'inst/unit':>9s} {'inst':>6s} {'samples':>7s}")
    for k, v in bi.most_common():
        print(f"  {k:28s} {v / float(units):9.0f} {v / ti:6.3f} {bs[k] / ts:7.3f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
