"""Key metrics + stall breakdown from an ncu report (dev aid): python scripts/ncu_summary.py rep.ncu-rep"""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print("kernel:", d.get("Kernel Name", "")[:100])
    keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "smsp__inst_executed.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
    for k in keys:
        if k in d:
            print(f"  {k:70s} {d[k]:>16s} {u.get(k, '')}")
    stalls = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled_") or
              k.startswith("smsp__pcsamp_warps_issue_stalled_")]
    st = []
    for k, v in stalls:
        try:
            st.append((float(v.replace(",", "")), k))
        except ValueError:
            pass
    for v, k in sorted(st, reverse=True)[:12]:
        print(f"  stall {k:80s} {v:g}")
