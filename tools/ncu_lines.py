"""Summarise an ncu source page (cuda,sass CSV) by CUDA source line:
instructions executed and stall samples per line, top N."""
import csv
import subprocess
import sys


def main(rep, kernel, top=30, which=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kernel}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    res = []
    fname = None
    func_count = -1
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] == "":
            continue
        try:
            ie = int(r[hdr.index("Instructions Executed")])
            smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        res.append((ie, smp, f"{fname}:{r[0]}", r[1].strip()[:90]))
    tot_i = sum(x[0] for x in res) or 1
    tot_s = sum(x[1] for x in res) or 1
    print(f"total instr {tot_i}  samples {tot_s}")
    for ie, smp, loc, s in sorted(res, key=lambda x: -x[1])[:top]:
        print(f"{ie / tot_i:6.3f} {smp / tot_s:6.3f} {loc:28s} {s}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30,
         int(sys.argv[4]) if len(sys.argv) > 4 else 0)
