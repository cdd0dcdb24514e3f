"""Brief of one kernel in an ncu report (development tool): duration, clocks, DRAM/L2/LSU/tensor
activity, issue-stall samples. python tools/ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units = r[0], r[1]
for v in r[2:]:
    d = dict(zip(h, v))
    print(d.get("Kernel Name", "")[:100])
    keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active"]
    for k in keys:
        if k in d:
            print(f"  {k} = {d[k]} {units[h.index(k)]}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k]) for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and d[k] not in ("", "n/a")}
    tot = sum(st.values()) or 1
    print("  stalls:", ", ".join(f"{k} {v / tot:.0%}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]))
