#!/bin/bash
# Round evidence for profiles/ (each ncu run only after the same command has
# exited 0 without ncu):
#   * ncu launch list of the headline bench command;
#   * per-config launch lists of one full ID (tools/prof_config.py);
#   * --set full captures of each config's dominant kernels.
# Then: python tools/make_profiles.py r02  (here, after the gpurun merge).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L="--metrics gpu__time_duration.sum --clock-control none --csv"
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-secondary"
$B > gpurun_out/pf_bench_plain.log 2>&1 && \
  ncu $L --log-file gpurun_out/pf_launches_bench.csv $B > gpurun_out/pf_ncu_bench.log 2>&1
for w in C2 C3 C4 C5; do
  python tools/prof_config.py --workload $w > gpurun_out/pf_plain_$w.log 2>&1 && \
    ncu $L --profile-from-start off --log-file gpurun_out/pf_launches_$w.csv \
      python tools/prof_config.py --workload $w \
      > gpurun_out/pf_ncu_$w.log 2>&1
done
full() {  # $1 kernel regex, $2 report name, $3.. prof_config args
  local k=$1 name=$2; shift 2
  ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:$k -s 1 -c 1 \
      -o gpurun_out/pf_full_$name python tools/prof_config.py "$@" > gpurun_out/pf_ncu_full_$name.log 2>&1
}
full cs_rowmajor cs_rowmajor --workload C2
full cs_coltile_ra cs_coltile_ra --workload C2 --fortran
full cs_csr_stream cs_csr_stream --workload C3
IDS_HASH_STAGES=1 full fy_phaseb fy_phaseb_c3 --workload C3
full cpqr_wide_kernel cpqr_wide_c3 --workload C3
full ts_split_kernel ts_split_c4 --workload C4
full ts_split_kernel ts_split_c5 --workload C5
full cpqr_tall_kernel cpqr_tall_c5 --workload C5
full cpqr_tall_kernel cpqr_tall_c4 --workload C4
echo profiles done
