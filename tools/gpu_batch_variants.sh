set -u
mkdir -p gpurun_out
for v in default b3 u2 u6; do
  if [ $v = default ]; then unset DAWN_LIB; else export DAWN_LIB=$PWD/paper_2306_07872_b200/libdawn_$v.so; fi
  echo "== $v"; timeout 300 python tools/apsp_probe.py --k 512 --single 4 > gpurun_out/c3_$v.txt 2>&1; head -1 gpurun_out/c3_$v.txt
done
unset DAWN_LIB
for o in degree random; do echo "== order $o"; timeout 300 python tools/apsp_probe.py --k 512 --single 4 --order $o 2>&1 | head -1; done
cat gpurun_out/c3_default.txt | tail -32
