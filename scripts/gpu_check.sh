#!/usr/bin/env bash
# gpurun helper: GPU tests (optionally a -k filter) + smoke + a short bench. Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
K=${K:-}
if [ -n "$K" ]; then
  timeout ${PT_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout ${PT_TIMEOUT:-1500} python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
if [ "${BENCH:-1}" = "1" ]; then
  timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
  tail -c 3000 gpurun_out/bench.log
fi
