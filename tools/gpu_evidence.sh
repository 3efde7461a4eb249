#!/bin/bash
# Evidence for profiles/: plain bench line, ncu launch list of the same bench
# command, and one full ncu capture of the dominant kernel (cs_rowmajor).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/ev_bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/ev_launches_bench.csv $CMD > gpurun_out/ev_ncu_bench.log 2>&1
python tools/prof_step.py --steps 1 > gpurun_out/ev_prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:cs_rowmajor -s 1 -c 1 \
      -o gpurun_out/ev_rowmajor python tools/prof_step.py --steps 1 > gpurun_out/ev_ncu_full.log 2>&1
echo evidence done
