#!/usr/bin/env bash
# A/B of library builds on the default bench: LIBS="name=path ..." (plus the product library as base),
# 2 alternating runs each; BENCH_ARGS passes extra bench flags.
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for spec in base= ${LIBS:-}; do
    name=${spec%%=*}; lib=${spec#*=}
    v=$(SPLATNAV_B200_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} 2>>gpurun_out/ab_err.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); s=d['stages_ms_per_step']; print(round(d['value']), d.get('render_retries'), {k: round(v, 3) for k, v in s.items() if k in ('scene.blend', 'layer.blend', 'layer.composite')})")
    echo "$name run$r: $v"
  done
done
