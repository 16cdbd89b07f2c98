mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_slicing.py -m gpu -x -q > gpurun_out/slicing.txt 2>&1; echo "slicing rc=$?"; tail -3 gpurun_out/slicing.txt
for r in 1 2; do for g in 0 1; do
v=$(SN_FAR_GRAPH=$g timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>>gpurun_out/ab_err.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); s=d['stages_ms_per_step']; print(round(d['value']), d.get('gpu_launches'), {k:round(v,3) for k,v in s.items() if 'far' in k or 'blend' in k})")
echo "graph=$g run$r: $v"
done; done
