"""Summarise an ncu --set full capture of one PCGM step (tools/ncu_step.sh) into
profiles/<round>/ncu_step_full_summary.json and profiles/ncu_traffic.json (DRAM bytes per
launch keyed by bench.py's kernel names): duration, DRAM and L2 traffic, HBM throughput, the
fp64 pipes (DFMA and the DMMA tensor subpipe), occupancy, issue activity and the stall mix.

    python tools/profile_summary.py gpurun_out/step_r02.ncu-rep profiles/r02
"""
import csv, io, json, os, subprocess, sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sectors_srcunit_tex.sum",
           "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def step_name(fn, seen):
    """Kernel function -> bench.py step-kernel name (launch order inside one step)."""
    if "k_dstep" in fn or "k_grid_r<0" in fn:
        return "delta"
    if "k_update_x" in fn:
        return "update_x"
    if "k_dirupdate_x" in fn:
        return "dirupdate_x"
    if "k_dirupdate" in fn:
        return "dirupdate"
    if "k_grid<3" in fn or "k_rstep" in fn:
        return "outer_rhs_s1"
    if "k_chainm<" in fn:   # k_chainm<NS, INNER, P, W, FR, DOT>
        targs = [x.strip() for x in fn.split("k_chainm<")[1].split(">")[0].split(",")]
        if targs[4] == "1":
            return "sweep_s0_l0_r"
        if targs[1] == "1":
            return "sweep_s0_l1" if "sweep_s0_l1" not in seen else "sweep_s1_l1"
        return "sweep_s1_l0"
    if "k_chain<2, 0, 7, 1, 0, 1" in fn:
        return "sweep_s0_l0_r"
    if "k_chain<2, 1" in fn:
        return "sweep_s0_l1" if "sweep_s0_l1" not in seen else "sweep_s1_l1"
    if "k_chain<2, 0" in fn:
        return "sweep_s1_l0"
    return fn[:40]


def main(rep, outdir):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out, traffic, seen = [], {}, set()
    for r in rows[2:]:
        fn = r[hdr.index("Kernel Name")]
        name = step_name(fn, seen)
        seen.add(name)
        rec = {"step_kernel": name, "function": fn}
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
            if h.startswith("smsp__average_warps_issue_stalled_") and \
                    h.endswith("_per_issue_active.ratio"):
                try:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(r[i])
                except ValueError:
                    pass
        rec["stalls_per_issue_top"] = dict(sorted(((k, round(v, 2)) for k, v in stalls.items()),
                                                  key=lambda kv: -kv[1])[:6])
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        u = units[hdr.index("dram__bytes_read.sum")]
        rec["dram_bytes"] = (rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]) * scale.get(u, 1.0)
        rec["l2_bytes_from_sm"] = rec["lts__t_sectors_srcunit_tex.sum"] * 32
        traffic.setdefault(name, rec["dram_bytes"])
        out.append(rec)
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, "ncu_step_full_summary.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    with open(os.path.join(os.path.dirname(outdir.rstrip("/")), "ncu_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    for rec in out:
        print(f"{rec['step_kernel']:14s} {rec['gpu__time_duration.sum']:8.1f} us  DRAM "
              f"{rec['dram_bytes'] / 1e6:7.1f} MB  L2<-SM {rec['l2_bytes_from_sm'] / 1e6:7.1f} MB  "
              f"fp64 {rec.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0):5.1f}%  "
              f"dmma {rec.get('sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active', 0):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
