#!/bin/bash
# Round-end evidence for profiles/: the bench line and its ncu launch list,
# per-config step launch lists (C2-C5), and --set full captures of the
# dominant kernel of each config (each ncu run only after the same command
# exited 0 without ncu).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/gpu_evidence.sh
EXTRA=1 bash tools/gpu_prof.sh
run_full() {  # $1 kernel regex, $2 report name, $3.. prof_step args
  local k=$1 name=$2; shift 2
  python tools/prof_step.py --steps 1 "$@" > gpurun_out/full_plain_$name.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 \
        -o gpurun_out/full_$name python tools/prof_step.py --steps 1 "$@" > gpurun_out/ncu_full_$name.log 2>&1
}
run_full tensorsketch_kernel tensorsketch_c5 --tensor 4,10000,2000,16384,20
run_full cpqr_kernel cpqr_c5 --tensor 4,10000,2000,16384,20
run_full cs_csr_stream cs_csr_stream --csr 10000000,10000,100000000,200,20
run_full fy_phaseb fy_phaseb
run_full cpqr_cluster cpqr_cluster
python tools/exp_fortran_one.py > gpurun_out/full_plain_coltile.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:cs_coltile -s 1 -c 1 \
      -o gpurun_out/full_cs_coltile python tools/exp_fortran_one.py > gpurun_out/ncu_full_coltile.log 2>&1
echo round profiles done
