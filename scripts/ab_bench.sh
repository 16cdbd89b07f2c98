#!/usr/bin/env bash
# A/B of library variants on the default bench: VARIANTS="name=path ..." (default lib = "base"), 2 runs each.
set -u
mkdir -p gpurun_out
for spec in base=paper_2604_12626_b200/libsplatnav_b200.so ${VARIANTS:-}; do
  name=${spec%%=*}; path=${spec#*=}
  for r in 1 2; do
    v=$(SPLATNAV_B200_LIB=$path timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} 2>>gpurun_out/ab_err.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['stages_ms_per_step'].get('scene.blend',0),3), round(d['stages_ms_per_step'].get('layer.blend',0),3))")
    echo "$name run$r: $v"
  done
done
