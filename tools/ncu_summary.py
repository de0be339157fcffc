"""Summarise an ncu --set full capture of the evaluation kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/<tag>_prof.ncu-rep profiles/<tag>_ncu [--launches launches.csv]

Writes <out>.json (machine-readable; bench.py reads dram_bytes_per_launch from
profiles/ncu_summary.json for roofline.traffic) and <out>.md (human-readable)."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_inst_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_inst_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_inst_executed",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefront_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma_thread",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd_thread",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul_thread",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "second": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    res = {"kernel": None, "launches": []}
    for v in vals:
        d = {"kernel": v[hdr.index("Kernel Name")]}
        for i, name in enumerate(hdr):
            if name in KEYS:
                try:
                    x = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                d[KEYS[name]] = x * UNIT.get(units[i], 1.0)
        res["launches"].append(d)
    L = res["launches"][0]
    res["kernel"] = L["kernel"]
    res["dram_bytes_per_launch"] = L.get("dram_read", 0) + L.get("dram_write", 0)
    res["stalls_per_issue"] = {}
    for i, name in enumerate(hdr):
        if name.startswith("smsp__average_warps_issue_stalled") and name.endswith("per_issue_active.ratio"):
            try:
                x = float(vals[0][i])
            except ValueError:
                continue
            if x >= 0.01:
                res["stalls_per_issue"][name.split("stalled_")[1].replace("_per_issue_active.ratio", "")] = x
    with open(out + ".json", "w") as fh:
        json.dump(res, fh, indent=1)
    with open(out + ".md", "w") as fh:
        fh.write(f"# ncu --set full summary: `{rep}`\n\nkernel: `{L['kernel']}`\n\n| metric | value |\n|---|---|\n")
        for k in KEYS.values():
            if k in L:
                fh.write(f"| {k} | {L[k]:.6g} |\n")
        fh.write(f"| dram_bytes_per_launch | {res['dram_bytes_per_launch']:.6g} |\n\n")
        fh.write("stall reasons (warps per issue, active):\n\n")
        for k, x in sorted(res["stalls_per_issue"].items(), key=lambda t: -t[1]):
            fh.write(f"- {k}: {x:.3f}\n")
    print(json.dumps({k: L.get(k) for k in ("duration", "fp64_pipe_active_pct", "issue_active_pct", "registers")}))


if __name__ == "__main__":
    main()
