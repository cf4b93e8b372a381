"""Summarise an ncu --set full report: key metrics, stall reasons, per-opcode samples/smem wavefronts."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.per_cycle_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]
for vals in rows[2:]:
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"{w:70s} {vals[i]:>24s} {units[i]}")
    st = [(h, vals[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio")]
    st = sorted(st, key=lambda x: -float(x[1] or 0))[:8]
    for h, v in st:
        print(f"  stall {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v}")
    try:
        dadd = float(vals[hdr.index("sm__sass_thread_inst_executed_op_dadd_pred_on.sum")].replace(",", ""))
        dmul = float(vals[hdr.index("sm__sass_thread_inst_executed_op_dmul_pred_on.sum")].replace(",", ""))
        dfma = float(vals[hdr.index("sm__sass_thread_inst_executed_op_dfma_pred_on.sum")].replace(",", ""))
        print(f"  executed FP64 flops (DADD+DMUL+2 DFMA) = {dadd + dmul + 2 * dfma:.6e}")
    except ValueError:
        pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
if len(srows) > 2:
    h = srows[1]
    I = h.index
    tot = sum(int(r[I("Warp Stall Sampling (All Samples)")] or 0) for r in srows[2:])
    byop, cnt, wf, wfi = collections.Counter(), collections.Counter(), collections.Counter(), collections.Counter()
    for r in srows[2:]:
        t = r[I("Source")].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        op = op.split(".")[0]
        byop[op] += int(r[I("Warp Stall Sampling (All Samples)")] or 0)
        cnt[op] += int(r[I("Instructions Executed")] or 0)
        try:
            wf[op] += int(r[I("L1 Wavefronts Shared")] or 0)
            wfi[op] += int(r[I("L1 Wavefronts Shared Ideal")] or 0)
        except ValueError:
            pass
    print(f"  stall samples: {tot}")
    for op, v in byop.most_common(12):
        print(f"  {op:8s} samples {100 * v / max(tot, 1):5.1f}%  warp-inst {cnt[op]:>12d}  smem wavefronts {wf[op]:>11d} (ideal {wfi[op]})")
