set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/bench_configs.py --solves 5 --out gpurun_out/configs.json > gpurun_out/configs.txt 2>&1; echo configs rc=$?
python -c "
import json
for l in open('gpurun_out/configs.txt'):
    if l.startswith('{'):
        r=json.loads(l); print(r['config'], 'jacobi', round(r['ms_median'],3), 'async', round(r['async_ms_median'],3), r['parity'])"
