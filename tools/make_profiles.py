"""Summaries for profiles/ from the ncu outputs of a gpurun (gpurun_out/).

usage: python tools/make_profiles.py ROUND   (e.g. r02), after tools/gpu_profiles.sh ran on the box

Writes, when the inputs exist:
  profiles/ROUND_bench_launches.csv          ncu launch list of the bench command
  profiles/ROUND_bench_launches_summary.txt  per-kernel counts / mean / total
  profiles/ROUND_step_launches_cN.txt        one countsketch_id / tensorsketch_id
                                             call per config (tools/prof_config.py)
  profiles/ROUND_<kernel>_ncu_full.txt       key metrics + top stall lines of the
                                             --set full captures
"""
import csv
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_sectors_srcunit_tex_op_red.sum",
    "lts__t_sectors_srcunit_tex_op_red_lookup_hit.sum",
    "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


def launches(src, dst, title):
    txt = run([sys.executable, os.path.join(ROOT, "tools", "launches.py"), src])
    with open(dst, "w") as fh:
        fh.write(f"# {title}\n# ncu --metrics gpu__time_duration.sum --clock-control none "
                 "(serialized, cold-cache per-launch times)\n")
        fh.write(txt)
    print("wrote", dst)


def full(rep, dst, title):
    raw = list(csv.reader(run(["ncu", "-i", rep, "--page", "raw", "--csv"]).splitlines()))
    if len(raw) < 3:
        return
    hdr, units, vals = raw[0], raw[1], raw[2]
    lines = [f"# {title}", f"# report: {os.path.relpath(rep, ROOT)}", ""]
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            lines.append(f"{m:70s} {vals[i]:>20s} {units[i]}")
    stalls = [(h, vals[i]) for i, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and vals[i].replace(".", "").isdigit()]
    stalls.sort(key=lambda t: -float(t[1]))
    lines += ["", "# top warp-stall reasons (samples)"]
    lines += [f"{h:70s} {v:>20s}" for h, v in stalls[:8]]
    hot = run([sys.executable, os.path.join(ROOT, "tools", "ncu_hot.py"), rep, "25", "cuda"])
    lines += ["", "# top CUDA source lines by warp-stall samples", hot]
    with open(dst, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("wrote", dst)


if os.path.exists(os.path.join(OUT, "pf_launches_bench.csv")):
    shutil.copy(os.path.join(OUT, "pf_launches_bench.csv"), os.path.join(PROF, f"{rnd}_bench_launches.csv"))
    launches(os.path.join(OUT, "pf_launches_bench.csv"), os.path.join(PROF, f"{rnd}_bench_launches_summary.txt"),
             "python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-secondary (whole process: "
             "data generation, warm-up, timed trials, roofline and phase timers)")
for cfg, what in (("C2", "C2 countsketch_id, dense 1e6 x 2000, K=20, L=100"),
                  ("C3", "C3 countsketch_id, CSR 1e7 x 1e4, ~1e8 nnz, K=20, L=200"),
                  ("C4", "C4 tensorsketch_id, N=3, I=1000, R=1000, K=10, L=4096"),
                  ("C5", "C5 tensorsketch_id, N=4, I=1e4, R=2000, K=20, L=16384")):
    src = os.path.join(OUT, f"pf_launches_{cfg}.csv")
    if os.path.exists(src):
        launches(src, os.path.join(PROF, f"{rnd}_step_launches_{cfg.lower()}.txt"),
                 f"{what}: tools/prof_config.py --workload {cfg} (warm-up call + one call)")
traffic = {}
for rep, name, title, key in (
        ("pf_full_cs_rowmajor.ncu-rep", "cs_rowmajor", "cs_rowmajor_kernel, C2 sketch (C order)", "C2"),
        ("pf_full_cs_coltile.ncu-rep", "cs_coltile", "cs_coltile_kernel (32-slot), C2 in F order", None),
        ("pf_full_cs_coltile_ra.ncu-rep", "cs_coltile_ra",
         "cs_coltile_ra_kernel<2,512,3> (bucket-sorted tiles, register accumulators), C2 in F order", None),
        ("pf_full_cs_csr_stream.ncu-rep", "cs_csr_stream", "cs_csr_stream_kernel, C3", "C3"),
        ("pf_full_fy_phaseb_c3.ncu-rep", "fy_phaseb_c3",
         "fy_phaseb_kernel, C3 hash (I = 1e7), the whole chain in one launch (ids_set_hash_stages(1))", None),
        ("pf_full_cpqr_wide_c3.ncu-rep", "cpqr_wide_c3",
         "cpqr_wide_kernel (column slices in shared memory), C3 sketch 200 x 10000, k = 20", None),
        ("pf_full_tensorsketch_c4.ncu-rep", "tensorsketch_c4", "tensorsketch_kernel<8>, C4", None),
        ("pf_full_tensorsketch_c5.ncu-rep", "tensorsketch_c5", "tensorsketch_kernel<16>, C5", None),
        ("pf_full_cpqr_c5.ncu-rep", "cpqr_c5", "cpqr_kernel, C5 sketch 16384 x 2000, k = 20", None),
        ("pf_full_ts_split_c4.ncu-rep", "ts_split_c4", "ts_split_kernel<1024> (split-spectrum TensorSketch), C4",
         "C4"),
        ("pf_full_ts_split_c5.ncu-rep", "ts_split_c5", "ts_split_kernel<4096> (split-spectrum TensorSketch), C5",
         "C5"),
        ("pf_full_cpqr_tall_c5.ncu-rep", "cpqr_tall_c5",
         "cpqr_tall_kernel (column-owning CPQR), C5 sketch 16384 x 2000, k = 20", None),
        ("pf_full_cpqr_tall_c4.ncu-rep", "cpqr_tall_c4",
         "cpqr_tall_kernel (column-owning CPQR), C4 sketch 4096 x 1000, k = 10", None)):
    p = os.path.join(OUT, rep)
    if os.path.exists(p):
        full(p, os.path.join(PROF, f"{rnd}_{name}_ncu_full.txt"), title)
        if key:
            raw = list(csv.reader(run(["ncu", "-i", p, "--page", "raw", "--csv"]).splitlines()))
            hdr, units, vals = raw[0], raw[1], raw[2]
            tot = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(m)
                tot += float(vals[i]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[i], 1)
            traffic[key] = tot
if traffic:
    import json

    tp = os.path.join(PROF, "traffic.json")
    t = json.load(open(tp)) if os.path.exists(tp) else {}
    t.update(traffic)
    t.update({"C2_bytes": 16_000_000_000, "C3_bytes": 1_239_938_912, "C4_bytes": 24_000_000,
              "C5_bytes": 640_000_000})
    t["_source"] = (f"profiles/{rnd}_*_ncu_full.txt: dram__bytes_read.sum + dram__bytes_write.sum "
                    "of one launch of each config's dominant kernel; <name>_bytes = the "
                    "algorithmic bytes of that launch")
    json.dump(t, open(tp, "w"), indent=1)
    print("wrote", tp, traffic)
