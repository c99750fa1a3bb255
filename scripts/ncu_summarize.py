"""Summarise an ncu --set full report into JSON: `ncu_summarize.py REP KEY [ROW]`
(ROW = index of the profiled launch in the report, default 0)."""
import csv
import io
import json
import subprocess
import sys

rep, key = sys.argv[1], sys.argv[2]
row = int(sys.argv[3]) if len(sys.argv) > 3 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2 + row]
m = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
SCALE = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def f(name):
    try:
        return float(m[name].replace(",", "")) * SCALE.get(u.get(name, ""), 1.0)
    except Exception:
        return None


dur_ns = f("gpu__time_duration.sum")  # seconds after unit scaling
rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
out = {key: {
    "kernel": m.get("Kernel Name", "")[:120],
    "duration_us": dur_ns * 1e6 if dur_ns else None,
    "dram_bytes_read": rd, "dram_bytes_write": wr,
    "dram_bytes_per_launch": (rd or 0) + (wr or 0),
    "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "sm_throughput_pct": f("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "fp64_pipe_active_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "ipc_active": f("sm__inst_executed.avg.per_cycle_active"),
    "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers": f("launch__registers_per_thread"),
    "grid": f("launch__grid_size"), "block": f("launch__block_size"),
    "smem_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "l2_hit_pct": f("lts__t_sector_hit_rate.pct"),
    "dfma_thread_inst": f("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"),
    "dadd_thread_inst": f("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"),
    "dmul_thread_inst": f("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"),
}}
print(json.dumps(out, indent=1))
