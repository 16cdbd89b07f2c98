#!/usr/bin/env bash
# A/B of an environment knob on the default bench: ENVS="name=VAR=value ..." (plus a plain base), 2 runs each.
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for spec in base=X=1 ${ENVS:-}; do
    name=${spec%%=*}; kv=${spec#*=}
    v=$(env "$kv" timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} 2>>gpurun_out/ab_err.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); s=d['stages_ms_per_step']; print(round(d['value']), d.get('gpu_launches'), d.get('render_retries'), {k: round(v, 3) for k, v in s.items() if k in ('scene.blend', 'scene.far', 'layer.blend')})")
    echo "$name run$r: $v"
  done
done
