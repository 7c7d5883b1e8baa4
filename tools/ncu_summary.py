"""Print the key metrics of `ncu --page raw --csv` exports (one launch each)."""
import csv, sys
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"), ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "inst executed"),
    ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__t_bytes.sum", "L1 bytes"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]
STALL = "smsp__average_warp_latency_issue_stalled_"
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
    print(f"== {path}: {d.get('Kernel Name', '')[:100]}")
    for k, name in KEYS:
        if k in d:
            print(f"  {name:16s} {d[k]} {u.get(k, '')}")
    st = [(k[len(STALL):].replace(".ratio", ""), float(d[k])) for k in hdr
          if k.startswith(STALL) and k.endswith(".ratio") and d[k] not in ("", "n/a")]
    st.sort(key=lambda t: -t[1])
    print("  stalls/issue:", ", ".join(f"{a} {b:.2f}" for a, b in st[:7]))
