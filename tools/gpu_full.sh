#!/bin/bash
# ncu --set full captures of named kernels of tools/prof_step.py (after a plain run).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python tools/prof_step.py --steps 1 $PROF_ARGS > gpurun_out/full_plain.log 2>&1 || exit 1
for K in $KERNELS; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-2} -c 1 \
      -o gpurun_out/full_$K python tools/prof_step.py --steps 1 $PROF_ARGS > gpurun_out/ncu_full_$K.log 2>&1
done
echo full done
