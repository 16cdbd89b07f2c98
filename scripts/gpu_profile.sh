#!/usr/bin/env bash
# Run on a B200 box via gpurun: the default bench, the ncu launch list of the same bench command,
# and one full ncu capture of the top kernels. Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
B="python bench.py"
timeout 900 $B > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
L="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$L > gpurun_out/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches.csv $L > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/ncu_launch.log
C="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$C > gpurun_out/plain_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"${NCU_REGEX:-blend_kernel<\(int\)0, \(int\)0>|blend_kernel_lp2|scene_emit|scene_count|avatar_count|avatar_emit|fixup_kernel<\(int\)0>}" -s ${NCU_SKIP:-21} -c ${NCU_COUNT:-8} -o gpurun_out/prof_full $C \
    > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
