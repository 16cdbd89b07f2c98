mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python scripts/sweep.py > gpurun_out/sweep_all.jsonl 2> gpurun_out/sweep_all.err
python -c "
import json
for l in open('gpurun_out/sweep_all.jsonl'):
    d=json.loads(l); s=d['stage_ms']; print(d.get('config'), d['n_gaussians'], d.get('n_avatars'), d.get('n_envs'), round(d['frames_per_s']), round(d['ms_per_step'],1), {k: round(v,1) for k,v in s.items() if v})
"; tail -2 gpurun_out/sweep_all.err
