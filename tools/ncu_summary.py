"""Summarise an ncu --set full report (and optionally a launch-list CSV) into profiles/."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
        "sm__cycles_active.max", "sm__cycles_elapsed.avg", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
        # FP64 tensor cores (DMMA): the pipe the direct core runs on
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg",
        "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {u[h.index(k)]}".strip()
        st = {n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: float(r[i])
              for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_")
              and n.endswith("_per_issue_active.ratio") and r[i] not in ("", "0")}
        d["stalls_per_issue"] = {k: v for k, v in sorted(st.items(), key=lambda x: -x[1]) if v > 0.05}
        res.append(d)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[1:]:
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        k = r[ik].split("(")[0]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    return {k: {"launches": a[0], "total": a[1], "share": round(a[1] / tot, 4)} for k, a in agg.items()}


if __name__ == "__main__":
    rep, out = sys.argv[1], sys.argv[2]
    d = {"ncu_full": raw(rep)}
    if len(sys.argv) > 3:
        d["launch_list"] = launches(sys.argv[3])
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d, indent=1)[:4000])
