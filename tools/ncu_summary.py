"""Key counters + stall reasons of one kernel in an ncu report.
usage: python tools/ncu_summary.py REPORT [KERNEL_REGEX]"""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'sm__inst_issued.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smsp__inst_executed.sum',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'launch__shared_mem_per_block_dynamic', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_bytes.sum']


def main(rep, kern=None):
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if kern:
        cmd += ["-k", "regex:" + kern]
    rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        print("==", v[h.index("Kernel Name")][:90])
        for k in KEYS:
            if k in h:
                print(f"  {k} {v[h.index(k)]} {units[h.index(k)]}")
        st = []
        for i, k in enumerate(h):
            if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
                try:
                    if float(v[i]) > 0:
                        st.append((float(v[i]), k.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1
        print("  stalls:", ", ".join(f"{n} {x / tot:.2f}" for x, n in sorted(st, reverse=True)[:8]))


if __name__ == "__main__":
    main(*sys.argv[1:])
