"""Write profiles/traffic.json (per-launch DRAM bytes, read + write) and, with a third
argument, profiles/round2_inst.json (per-launch warp instructions executed,
smsp__inst_executed.sum, with the units one launch processes) of each hot-path kernel from an
ncu --set full capture of tools/prof_driver.py at the bench's sizes.
usage: python tools/traffic_from_ncu.py REPORT traffic.json [inst.json]"""
import csv
import json
import subprocess
import sys

NAMES = {"grid_kernel": "eval_grid", "list_kernel": "eval_list", "radius_kernel": "profile_radius",
         "cluster_kernel": "profile_cluster", "cluster2_kernel": "profile_cluster"}
UNITS = {"eval_grid": 65536, "eval_list": 65536, "profile_radius": 65536, "profile_cluster": 65536,
         "thief_steepest": 65536, "thief_literal": 65536}


def main(rep, out, inst_out=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    res, ins = {}, {}
    thief = 0
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "inst": 1, "Kinst": 1e3,
             "Minst": 1e6, "Ginst": 1e9}
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
        if key is None or key in res:
            continue
        val = lambda m: float(d[m].replace(",", "")) * scale.get(u[m], 1)
        res[key] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        if d.get("smsp__inst_executed.sum"):
            ins[key] = {"warp_inst_per_launch": val("smsp__inst_executed.sum"), "units": UNITS[key],
                        "source": f"ncu smsp__inst_executed.sum, {rep.split('/')[-1]}"}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    if inst_out:
        with open(inst_out, "w") as f:
            json.dump(ins, f, indent=1)
    print(json.dumps(res, indent=1), json.dumps(ins, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
