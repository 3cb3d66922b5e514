"""Stall-reason and pipe summary of ncu reports: ncu_stalls.py rep1 [rep2 ...]."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"]
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units, v = r[0], r[1], r[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    print(f"== {rep}")
    for k in KEYS:
        if k in d:
            print(f"  {k:80s} {d[k]} {u[k]}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(x.replace(",", ""))
          for k, x in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("not_issued") and x}
    tot = sum(st.values())
    print("  stall samples: " + ", ".join(f"{k} {100 * x / tot:.1f}%" for k, x in
                                         sorted(st.items(), key=lambda t: -t[1]) if x / tot > 0.005))
