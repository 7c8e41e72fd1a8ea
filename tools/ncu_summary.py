"""Summarise an .ncu-rep (read here, no GPU): key metrics per kernel launch -> JSON.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [out.json]
"""
import csv, io, json, subprocess, sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "registers",
    "launch__occupancy_limit_registers": "occ_limit_registers_blocks",
    "sm__warps_active.avg.per_cycle_active": "warps_active_per_sm",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_inst",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_inst_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_inst_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_inst_pct",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum": "ffma",
    "sm__sass_thread_inst_executed_op_fadd_pred_on.sum": "fadd",
    "sm__sass_thread_inst_executed_op_fmul_pred_on.sum": "fmul",
    "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum": "local_ld_bytes",
    "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum": "local_st_bytes",
}
STALL = "smsp__average_warps_issue_stalled_"


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for vals in data:
        d = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for i, h in enumerate(hdr):
            if h in KEYS:
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u == "Gbyte": v *= 1e9
                elif u == "Mbyte": v *= 1e6
                elif u == "Kbyte": v *= 1e3
                elif u == "ms": v *= 1e-3
                elif u == "us": v *= 1e-6
                elif u == "ns": v *= 1e-9
                d[KEYS[h]] = v
            elif h.startswith(STALL) and h.endswith("_per_issue_active.ratio"):
                try:
                    d.setdefault("stalls", {})[h[len(STALL):-len("_per_issue_active.ratio")]] = float(vals[i])
                except ValueError:
                    pass
        if "stalls" in d:
            d["stalls"] = dict(sorted(d["stalls"].items(), key=lambda kv: -kv[1])[:8])
        out.append(d)
    return out


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    txt = json.dumps(res, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(txt)
    print(txt)
