"""Write profiles/traffic.json: per-launch DRAM bytes (read + write) of each hot-path
kernel from an ncu --set full capture of tools/prof_driver.py at the bench's sizes."""
import csv
import json
import subprocess
import sys

NAMES = {"grid_kernel": "eval_grid", "list_kernel": "eval_list", "radius_kernel": "profile_radius",
         "cluster_kernel": "profile_cluster"}


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    res = {}
    thief = 0
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        name = d["Kernel Name"]
        key = None
        for k, v in NAMES.items():
            if k in name:
                key = v
        if "thief_kernel" in name:
            key = ["thief_steepest", "thief_literal"][thief % 2]
            thief += 1
        if key is None:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        rd = float(d["dram__bytes_read.sum"]) * scale.get(u["dram__bytes_read.sum"], 1)
        wr = float(d["dram__bytes_write.sum"]) * scale.get(u["dram__bytes_write.sum"], 1)
        res[key] = rd + wr
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
