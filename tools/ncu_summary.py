"""Summarise an ncu --set full report into a small JSON for profiles/ (tooling).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/out.json "note"
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep, out, note=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    kernels = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")][:160]}
        for i, name in enumerate(h):
            if name in KEYS:
                d[name] = f"{v[i]} {units[i]}".strip()
        stalls = {}
        for i, name in enumerate(h):
            if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
                try:
                    stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["stall_pct_of_samples"] = {k: round(100 * x / tot, 2)
                                     for k, x in sorted(stalls.items(), key=lambda t: -t[1]) if x / tot > 0.002}
        kernels.append(d)
    json.dump({"report": rep, "note": note, "kernels": kernels}, open(out, "w"), indent=1)
    print(json.dumps(kernels[0], indent=1)[:1500])


if __name__ == "__main__":
    main(*sys.argv[1:])
