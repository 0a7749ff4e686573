"""Summarise an ncu --set full report (per launch): duration, DRAM bytes, SM / memory
throughput, tensor-pipe utilisation (tcgen05: sm__pipe_tensor_cycles_active_realtime,
sm__mem_tensor_cycles_active = TMEM traffic), grid, registers, achieved occupancy.
Diagnostic (writes CSV to stdout)."""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__cycles_active.avg", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
     "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
     "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "launch__grid_size", "launch__registers_per_thread",
     "sm__warps_active.avg.pct_of_peak_sustained_active"]
rep = sys.argv[1]
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"]).decode()
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
w = csv.writer(sys.stdout)
cols = [m for m in M if m in hdr]
w.writerow(["ID", "kernel"] + [f"{m} [{units[hdr.index(m)]}]" for m in cols])
for r in rows[2:]:
    w.writerow([r[hdr.index("ID")], r[hdr.index("Kernel Name")][:60]] + [r[hdr.index(m)] for m in cols])
