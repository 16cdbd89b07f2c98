#!/usr/bin/env bash
# A/B of library variants at BASELINE config 4 (3M scene, 1,024 envs) with A avatars: VARIANTS="name=path ..."
set -u
mkdir -p gpurun_out
A=${A:-16}
for spec in base=paper_2604_12626_b200/libsplatnav_b200.so ${VARIANTS:-}; do
  name=${spec%%=*}; path=${spec#*=}
  SPLATNAV_B200_LIB=$path timeout 900 python bench.py --config 4 --avatars $A --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/c4_$name.log 2>>gpurun_out/ab_err.log
  python -c "import json; d=json.loads(open('gpurun_out/c4_$name.log').readline()); s=d['stages_ms_per_step']; print('$name', round(d['value']), {k: round(v,1) for k,v in s.items() if v > 2})"
done
