#!/bin/bash
# One GPU round trip: parity tests, bench, launch list, ncu captures of the
# persistent single-source kernel (C2) and the batched kernel (C3), per-round
# timelines.  Run under gpurun from the repo root:
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [tests|bench|ncu|ncu_c2|ncu_batch|all]'
# (ncu = both captures; together they can exceed gpurun's 64 MiB return limit)
set -u
what=${1:-all}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [[ $what == all || $what == tests ]]; then
  timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
fi
if [[ $what == all || $what == bench ]]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"; tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
  timeout 600 python tools/round_profile.py --solves 5 --out gpurun_out/rounds_c2.json > gpurun_out/rounds_c2.txt 2>&1
  timeout 600 python tools/round_profile.py --solves 5 --schedule jacobi > gpurun_out/rounds_c2_jacobi.txt 2>&1
  timeout 600 python tools/apsp_probe.py --k 512 --single 8 > gpurun_out/rounds_c3.txt 2>&1
fi
if [[ $what == all || $what == ncu || $what == ncu_c2 ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --apsp-sources 256 > gpurun_out/ncu_bench.log 2>&1
  echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dawn_persistent -s 2 -c 1 \
    -o gpurun_out/prof_c2 -f python tools/round_profile.py --solves 3 > gpurun_out/ncu_full.log 2>&1
  echo "ncu c2 rc=$?"
fi
if [[ $what == ncu_wl ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dawn_worklist -s 2 -c 1 \
    -o gpurun_out/prof_wl -f python tools/round_profile.py --solves 3 > gpurun_out/ncu_wl.log 2>&1
  echo "ncu worklist rc=$?"
fi
if [[ $what == all || $what == ncu || $what == ncu_batch ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dawn_batch_persistent -s 3 -c 1 \
    -o gpurun_out/prof_batch -f python tools/apsp_probe.py --k 128 --single 2 > gpurun_out/ncu_batch.log 2>&1
  echo "ncu batch rc=$?"
fi
