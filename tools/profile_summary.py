"""Summarise an ncu --set full capture of one PCGM step into profiles/<round>/ and
profiles/ncu_traffic.json (dram bytes per launch, keyed by the bench's kernel names).

    python tools/profile_summary.py gpurun_out/r01/step_full.ncu-rep profiles/r01
"""
import csv, io, json, os, subprocess, sys

# one PCGM step as captured by tools/stepprof.py (launch order); the first outer sweep
# carries the fused r update (sweep_s0_l0_r)
STEP_NAMES = ["delta", "update_x", "sweep_s0_l0_r", "sweep_s0_l1", "outer_rhs_s1",
              "sweep_s1_l0", "sweep_s1_l1", "dirupdate"]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
           "smsp__inst_executed_pipe_fp64.sum", "lts__t_sector_hit_rate.pct"]


def main(rep, outdir):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out, traffic = [], {}
    for k, r in enumerate(rows[2:]):
        rec = {"step_kernel": STEP_NAMES[k] if k < len(STEP_NAMES) else f"k{k}",
               "function": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                v = r[hdr.index(m)]
                try:
                    v = float(v.replace(",", ""))
                except ValueError:
                    pass
                rec[m] = v
                rec[m + ".unit"] = units[hdr.index(m)]
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(r[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        rec["stall_pct_top"] = dict(sorted(((k2, round(100 * v / tot, 1)) for k2, v in stalls.items()),
                                           key=lambda kv: -kv[1])[:6])
        scale = 1e6 if units[hdr.index("dram__bytes_read.sum")].startswith("M") else \
            1e9 if units[hdr.index("dram__bytes_read.sum")].startswith("G") else 1.0
        rec["dram_bytes"] = (rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]) * scale
        traffic.setdefault(rec["step_kernel"], rec["dram_bytes"])
        out.append(rec)
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, "ncu_step_full_summary.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    tp = os.path.join(os.path.dirname(outdir.rstrip("/")), "ncu_traffic.json")
    with open(tp, "w") as fh:
        json.dump(traffic, fh, indent=1)
    for rec in out:
        print(rec["step_kernel"], rec["function"][:40], rec.get("gpu__time_duration.sum"),
              rec["dram_bytes"] / 1e6, "MB", rec["stall_pct_top"])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
