set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_nearfar.py -x -q > gpurun_out/nf_tests.log 2>&1; echo "nf tests rc=$?"; tail -3 gpurun_out/nf_tests.log
for pc in 4,64 2,16; do timeout 300 python tools/nearfar_probe.py --grid 4096 --profile $pc; done
timeout 900 python tools/nearfar_probe.py --grid 4096 --means 1,2,4,8 --caps 8,16,64 --solves 2 > gpurun_out/nf_g4096.txt 2>&1; echo g4096 rc=$?; cat gpurun_out/nf_g4096.txt | cut -c1-200
