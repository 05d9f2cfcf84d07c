"""Summarise a round's GPU evidence into profiles/: the ncu launch list (per-kernel ms and
share of the step), key counters of one --set full capture per hot kernel, DRAM traffic per
launch (profiles/traffic.json, read by bench.py) and the bench line.
usage: python tools/profile_summary.py EVIDENCE_DIR TAG"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the bench's A1 launch: cluster2_kernel computes both estimates (fused); older captures ran
# CLUSTER alone (PROFILE_ROW=profile_cluster)
NAMES = [("cluster2_kernel", os.environ.get("PROFILE_ROW", "profile")), ("cluster_kernel", "profile_cluster"),
         ("radius_kernel", "profile_radius"), ("grid_kernel", "eval_grid"), ("list_kernel", "eval_list"), ("list2_kernel", "eval_list"),
         ("thief_kernel<0", "thief_steepest"), ("thief_kernel<1", "thief_literal"),
         ("curve_fit_kernel", "next2_curve_fit"), ("uniform_kernel", "next3_uniform"),
         ("pareto_kernel", "next3_pareto"), ("prune_", "next3_prune"), ("place_kernel", "next4_placement"),
         ("checkpoint_kernel", "next4_checkpoint")]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def row_name(kernel, thief_seen):
    for k, v in NAMES:
        if k in kernel:
            return v
    if "thief_kernel" in kernel:
        return ["thief_steepest", "thief_literal"][thief_seen % 2]
    return None


def main(ev, tag):
    out_dir = os.path.join(ROOT, "profiles")
    # launch list
    rows = []
    with open(os.path.join(ev, "launches.csv")) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"]) / 1e6))
    tot = sum(ms for _, ms in rows) or 1
    per = {}
    for k, ms in rows:
        n = row_name(k, 0) or k[:40]
        if "thief_kernel" in k and n is None:
            n = "thief"
        per.setdefault(n, []).append(ms)
    # full capture
    txt = subprocess.run(["ncu", "-i", os.path.join(ev, "full.ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    fr = list(csv.reader(txt.splitlines()))
    h, units = fr[0], fr[1]
    full, traffic, insts = [], {}, {}
    thief = 0
    for r in fr[2:]:
        d = dict(zip(h, r))
        name = row_name(d["Kernel Name"], thief)
        if "thief_kernel" in d["Kernel Name"] and "<" not in d["Kernel Name"]:
            thief += 1
        u = dict(zip(h, units))
        rd = float(d["dram__bytes_read.sum"]) * SCALE.get(u["dram__bytes_read.sum"], 1)
        wr = float(d["dram__bytes_write.sum"]) * SCALE.get(u["dram__bytes_write.sum"], 1)
        if name:
            traffic[name] = rd + wr
            ie = d.get("smsp__inst_executed.sum", "")
            if ie:
                ie = float(ie) * {"inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}.get(
                    u.get("smsp__inst_executed.sum", "inst"), 1)
                # prof_driver.py launches every row at the bench sizes: 65,536 instances / queries
                insts[name] = {"warp_inst_per_launch": ie, "units": 65536,
                               "source": f"ncu --set full, smsp__inst_executed.sum ({tag})"}
        full.append((name or d["Kernel Name"][:40], {k: (d.get(k, ""), u.get(k, "")) for k in KEYS}))
    with open(os.path.join(out_dir, "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    with open(os.path.join(out_dir, "round2_inst.json"), "w") as f:
        json.dump(insts, f, indent=1)
    with open(os.path.join(out_dir, f"{tag}_ncu_full_summary.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["row"] + KEYS)
        for n, d in full:
            w.writerow([n] + [f"{v} {u}".strip() for v, u in d.values()])
    # the JSON line (a library banner may precede it in older captures)
    with open(os.path.join(ev, "bench.json")) as f:
        bench = json.loads([ln for ln in f if ln.startswith("{")][-1])
    with open(os.path.join(out_dir, f"{tag}_bench.json"), "w") as f:
        json.dump(bench, f, indent=1)
    md = [f"# {tag}: launch list, ncu counters, bench line\n",
          "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` of "
          "`python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-context` "
          f"(`{tag}_launches.csv`; cold-cache, serialised: compare shares).  Counters: one "
          "`ncu --set full --clock-control none --import-source on` capture per kernel of "
          f"`tools/prof_driver.py` at the bench sizes (`{tag}_ncu_full_summary.csv`).  Bench line: "
          f"`{tag}_bench.json`.\n",
          "| row | ncu ms/launch | ncu share | bench ms/launch | bench share | DRAM GB/launch | issue active % | warps active % |",
          "|---|---|---|---|---|---|---|---|"]
    step_ms = bench["ms_per_step"]
    fd = {n: d for n, d in full}
    for n in ["profile", "profile_cluster", "profile_radius", "eval_grid", "eval_list", "thief_steepest", "thief_literal",
              "next2_curve_fit", "next3_uniform", "next3_pareto", "next3_prune", "next4_placement", "next4_checkpoint"]:
        ms = per.get(n, [])
        nm = sum(ms) / len(ms) if ms else float("nan")
        share = sum(ms) / tot if ms else float("nan")
        b = bench["rows"].get(n, bench.get("context", {}).get(n, {}))
        d = fd.get(n, {})
        g = traffic.get(n, float("nan")) / 1e9
        bms = b.get("ms_per_launch", b.get("ms", float("nan")))
        md.append(f"| {n} | {nm:.3f} | {share:.3f} | {bms:.3f} | "
                  f"{b.get('share', float('nan')):.3f} | {g:.2f} | "
                  f"{d.get('sm__inst_issued.avg.pct_of_peak_sustained_active', ('',))[0]} | "
                  f"{d.get('sm__warps_active.avg.pct_of_peak_sustained_active', ('',))[0]} |")
    md.append("")
    md.append(f"Bench: value {bench['value']:.4g} {bench['unit']}, {step_ms:.2f} ms/step, clocks {bench['clocks']}; "
              f"roofline ({bench['roofline']['kernel']}): {bench['roofline']['achieved']:.2f} of "
              f"{bench['roofline']['peak']:.1f} {bench['roofline']['unit']} = {bench['roofline']['frac']:.3f}.")
    md.append("")
    md.append("Per-row roofline fractions (bench, CUDA events): " + ", ".join(
        (f"{k} {v['alu_frac']:.3f} (alu)" if "alu_frac" in v else f"{k} {v['hbm_frac']:.3f} (hbm)"
         if "hbm_frac" in v else f"{k} {v['issue_frac']:.3f} (issue)" if "issue_frac" in v else f"{k} -")
        for k, v in bench["rows"].items()))
    with open(os.path.join(out_dir, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    subprocess.run(["cp", os.path.join(ev, "launches.csv"), os.path.join(out_dir, f"{tag}_launches.csv")])
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
