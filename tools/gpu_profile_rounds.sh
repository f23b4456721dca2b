set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python tools/bench_configs.py --solves 5 --out gpurun_out/configs.json > gpurun_out/configs.txt 2>&1; echo configs rc=$?
timeout 300 python tools/round_profile.py --scale 14 --ef 8 --weights int --precision auto --solves 3 --schedule jacobi > gpurun_out/rounds_c1_jacobi.txt 2>&1; echo c1 rc=$?
timeout 300 python tools/round_profile.py --scale 14 --ef 8 --weights int --precision auto --solves 3 --schedule async > gpurun_out/rounds_c1_async.txt 2>&1
timeout 600 python tools/round_profile.py --grid 4096 --precision auto --solves 1 --schedule jacobi > gpurun_out/rounds_c4.txt 2>&1; echo c4 rc=$?
timeout 600 python tools/round_profile.py --solves 3 > gpurun_out/rounds_c2.txt 2>&1; echo c2 rc=$?
