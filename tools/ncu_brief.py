"""Key counters + stall reasons per kernel from an ncu report (raw page CSV)."""
import csv, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__waves_per_multiprocessor", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    print(r[hdr.index("Kernel Name")])
    print("   " + ", ".join(f"{w.split('__')[1][:40]}={r[hdr.index(w)]}" for w in want if w in hdr))
    st = [(hdr[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(r[i] or 0))
          for i in range(len(hdr)) if hdr[i].startswith("smsp__average_warps_issue_stalled")]
    st.sort(key=lambda x: -x[1])
    print("   stalls: " + ", ".join(f"{h}={v:.2f}" for h, v in st[:6]))
