"""Key metrics of every kernel in an ncu report (read here, no GPU):
    python tools/ncu_brief.py gpurun_out/x.ncu-rep"""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_srcunit_tex.sum", "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(r[hdr.index("Kernel Name")][:90])
        for k in KEYS:
            if k in hdr:
                print(f"   {k:78s} {r[hdr.index(k)]:>14s} {units[hdr.index(k)]}")
        st = {h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: float(r[i] or 0)
              for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
              and h.endswith("_per_issue_active.ratio")}
        top = sorted(st.items(), key=lambda kv: -kv[1])[:7]
        print("   stalls/issue:", ", ".join(f"{k} {v:.2f}" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
