#!/bin/bash
# Per-kernel launch lists (ncu, serialized cold-cache times) for the C2 matrix
# step and the C4 tensor step, plus one full capture of the sketch kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum --clock-control none --csv"
python tools/prof_step.py --steps 1 > gpurun_out/prof_c2_plain.log 2>&1 && \
  ncu $M --log-file gpurun_out/launches_c2.csv python tools/prof_step.py --steps 1 > gpurun_out/ncu_c2.log 2>&1
python tools/prof_step.py --steps 1 --tensor 3,1000,1000,4096,10 > gpurun_out/prof_c4_plain.log 2>&1 && \
  ncu $M --log-file gpurun_out/launches_c4.csv python tools/prof_step.py --steps 1 --tensor 3,1000,1000,4096,10 > gpurun_out/ncu_c4.log 2>&1
if [ -n "$FULL_KERNEL" ]; then
  ncu --set full --clock-control none --import-source on -k regex:$FULL_KERNEL -s ${FULL_SKIP:-1} -c 1 \
      -o gpurun_out/prof_full python tools/prof_step.py --steps 1 $FULL_ARGS > gpurun_out/ncu_full.log 2>&1
fi
echo "prof done"
if [ -n "$EXTRA" ]; then
python tools/prof_step.py --steps 1 --tensor 4,10000,2000,16384,20 > gpurun_out/prof_c5_plain.log 2>&1 && \
  ncu $M --log-file gpurun_out/launches_c5.csv python tools/prof_step.py --steps 1 --tensor 4,10000,2000,16384,20 > gpurun_out/ncu_c5.log 2>&1
python tools/prof_step.py --steps 1 --csr 10000000,10000,100000000,200,20 > gpurun_out/prof_c3_plain.log 2>&1 && \
  ncu $M --log-file gpurun_out/launches_c3.csv python tools/prof_step.py --steps 1 --csr 10000000,10000,100000000,200,20 > gpurun_out/ncu_c3.log 2>&1
echo extra done
fi
