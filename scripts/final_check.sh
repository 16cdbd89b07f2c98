#!/usr/bin/env bash
# Round-end evidence on one B200 (gpurun): GPU suite plain and bounds-checked, smoke, the reference
# arm, then scripts/gpu_profile.sh (bench line, ncu launch list, ncu --set full of the top kernels).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
SPLATNAV_B200_LIB=build_variants/libsn_checks.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_checks.log 2>&1; echo "checks rc=$?" >> gpurun_out/pytest_gpu_checks.log; tail -2 gpurun_out/pytest_gpu_checks.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "reference rc=$?" >> gpurun_out/bench_reference.log; tail -c 600 gpurun_out/bench_reference.log
bash scripts/gpu_profile.sh
tail -c 1500 gpurun_out/bench.log; tail -n 2 gpurun_out/ncu_launch.log; tail -n 2 gpurun_out/ncu_full.log
