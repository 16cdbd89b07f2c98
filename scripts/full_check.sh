mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
SPLATNAV_B200_LIB=build_variants/libsn_checks.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_checks.log 2>&1; echo "checks rc=$?" >> gpurun_out/pytest_gpu_checks.log; tail -3 gpurun_out/pytest_gpu_checks.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; tail -c 1500 gpurun_out/bench.log
