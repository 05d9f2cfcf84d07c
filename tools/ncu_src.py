"""Per-source-line instruction / stall-sample breakdown of one kernel in an ncu report.
usage: python tools/ncu_src.py REPORT KERNEL_REGEX UNITS [TOP]"""
import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, kern, units, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    res, smp = {}, {}
    fname, hdr = None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] == "" or hdr is None:
            continue
        try:
            ie = int(r[hdr.index("Instructions Executed")])
            sm = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        k = (fname, int(r[0]))
        res[k] = res.get(k, 0) + ie
        smp[k] = smp.get(k, 0) + sm
    tot = sum(res.values()) or 1
    ts = sum(smp.values()) or 1
    print(f"instructions per unit {tot / units:.0f}")
    cache = {}
    key = (lambda x: -smp[x[0]]) if os.environ.get("BY_SAMPLES") else (lambda x: -x[1])
    for (f, l), v in sorted(res.items(), key=key)[:top]:
        if f not in cache:
            cache[f] = open(f).read().split("\n") if os.path.exists(f) else []
        t = cache[f][l - 1].strip()[:80] if l - 1 < len(cache[f]) else ""
        print(f"{v / tot:6.3f} {smp[(f, l)] / ts:6.3f} {os.path.basename(f)}:{l} {t}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 30)
