#!/bin/bash
# One GPU session: environment facts, tests, smoke, a short bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{ nvidia-smi; free -g; nproc; python -c "import torch;print(torch.__version__, torch.cuda.get_device_name(0))"; } > gpurun_out/env.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
if [ -n "$BENCH_ARGS" ]; then
  timeout 900 python bench.py $BENCH_ARGS > gpurun_out/bench.log 2>&1
  echo "bench exit $?" >> gpurun_out/bench.log
fi
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log; tail -3 gpurun_out/bench.log 2>/dev/null
