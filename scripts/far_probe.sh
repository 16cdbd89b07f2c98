mkdir -p gpurun_out
SPLATNAV_B200_LIB=$PWD/build_variants/libsn_checks.so timeout 900 python -m pytest tests/test_slicing.py -q > gpurun_out/pt_slicing_chk.log 2>&1; tail -2 gpurun_out/pt_slicing_chk.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > gpurun_out/b.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.log').readline()); print(round(d['value']), d['render_retries'], {k: round(v,3) for k,v in d.get('stages_ms_per_step',{}).items() if k.startswith('scene')})"
timeout 900 python scripts/sweep.py config3 > gpurun_out/sw3.jsonl 2> gpurun_out/sw3.err
python -c "
import json
for l in open('gpurun_out/sw3.jsonl'):
    d=json.loads(l); s=d['stage_ms']; print(d['n_gaussians'], round(d['frames_per_s']), round(d['ms_per_step'],1), {k: round(v,1) for k,v in s.items() if v})
"; tail -2 gpurun_out/sw3.err
