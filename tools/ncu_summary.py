"""Key metrics of the first kernel in an ncu report (raw page)."""
import csv
import io
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, vals = rows[0], rows[2]
d = dict(zip(hdr, vals))
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"]
for k in keys:
    if k in d:
        print(f"{k:70s} {d[k]}")
stalls = {k: float(v) for k, v in d.items()
          if re.search(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$", k) and not k.endswith("not_issued")
          and v.replace(".", "").isdigit()}
tot = sum(stalls.values()) or 1
for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {v / tot * 100:5.1f}%")
