set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_worklist.py -x -q 2>&1 | tail -2
timeout 300 python tools/round_profile.py --scale 14 --ef 8 --weights int --precision auto --solves 5 --schedule jacobi 2>&1 | head -14
timeout 300 python tools/round_profile.py --solves 5 2>&1 | head -18
timeout 600 python tools/bench_configs.py --only c1,c2,c5a --solves 7 > gpurun_out/configs.txt 2>&1
python -c "
import json
for l in open('gpurun_out/configs.txt'):
    if l.startswith('{'):
        r=json.loads(l); print(r['config'], 'jacobi', round(r['ms_median'],4), 'async', round(r['async_ms_median'],4), all(v for v in r['parity'].values() if isinstance(v,bool)))"
