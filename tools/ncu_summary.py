"""Key metrics of ncu reports as JSON (for profiles/).  usage: ncu_summary.py rep..."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__inst_executed_pipe_fp64.sum": "fp64_warp_instructions",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}
out = {}
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")]
        d = {}
        for k, short in KEYS.items():
            if k in h:
                i = h.index(k)
                d[short] = f"{v[i]} {u[i]}".strip()
        out[f"{rep}:{name}"] = d
print(json.dumps(out, indent=1))
