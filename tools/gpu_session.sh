#!/bin/bash
# One GPU session: build check, tests (optionally filtered), smoke, bench.
#   PYTEST_K="config or cpqr" BENCH_ARGS="--steps 10 --warmup 3" tools/gpu_session.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{ nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; nproc; free -g; } > gpurun_out/env.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 ${PYTEST_K:+-k "$PYTEST_K"} ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  echo "smoke exit $?" >> gpurun_out/smoke.log
fi
if [ -n "$BENCH_ARGS" ]; then
  timeout 1200 python bench.py $BENCH_ARGS > gpurun_out/bench.log 2>&1
  echo "bench exit $?" >> gpurun_out/bench.log
fi
if [ -n "$EXTRA" ]; then
  bash -c "$EXTRA" > gpurun_out/extra.log 2>&1
  echo "extra exit $?" >> gpurun_out/extra.log
fi
tail -15 gpurun_out/pytest_gpu.log 2>/dev/null; tail -3 gpurun_out/smoke.log 2>/dev/null; tail -c 3000 gpurun_out/bench.log 2>/dev/null; tail -20 gpurun_out/extra.log 2>/dev/null
true
