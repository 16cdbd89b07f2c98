#!/usr/bin/env bash
# A/B: the in-tree library vs VARIANTS="name=path ..." on the default bench (2 runs each, interleaved),
# optional GPU tests first (TESTS="pytest args").
set -u
mkdir -p gpurun_out
if [ -n "${TESTS:-}" ]; then
  timeout 1500 python -m pytest ${TESTS} -q -x > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_tests.log
fi
for r in 1 2; do
  for spec in base=paper_2604_12626_b200/libsplatnav_b200.so ${VARIANTS:-}; do
    name=${spec%%=*}; path=${spec#*=}
    v=$(SPLATNAV_B200_LIB=$path timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} 2>>gpurun_out/ab_err.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); s=d['stages_ms_per_step']; print(round(d['value']), {k: round(v, 3) for k, v in s.items() if k in ('scene.blend', 'layer.count', 'layer.emit', 'layer.blend', 'scene.count')})")
    echo "$name run$r: $v"
  done
done
