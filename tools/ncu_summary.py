"""Summarise an `ncu --set full` report into the plain-text form kept under profiles/.

Usage: python tools/ncu_summary.py REPORT.ncu-rep "header line" [> profiles/rNN_....txt]
Also prints, on stderr, the JSON that bench.py reads for roofline.traffic (first wf_isect<.., 0>
launch: dram read + write bytes per launch)."""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_warps_issue_stalled_dispatch_stall", "smsp__pcsamp_warps_issue_stalled_branch_resolving",
]


def main():
    rep, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    idx = {n: i for i, n in enumerate(head)}
    print(header)
    traffic = None
    for r in data:
        name = r[idx["Kernel Name"]]
        print(f"\n## [{r[idx['ID']]}] {name}")
        for m in METRICS:
            if m in idx:
                print(f"{m:<82} {r[idx[m]]} {units[idx[m]]}")
        if traffic is None and "wf_isect<1, 0>" in name:
            def b(m):
                v = float(r[idx[m]].replace(",", ""))
                u = units[idx[m]]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            traffic = b("dram__bytes_read.sum") + b("dram__bytes_write.sum")
    if traffic is not None:
        print(json.dumps({"kernel": "wf_isect<smem, closest>", "dram_bytes_per_launch": traffic,
                          "source": rep}), file=sys.stderr)


if __name__ == "__main__":
    main()
