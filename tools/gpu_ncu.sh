set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
tag=${1:-r02}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --apsp-sources 256 > gpurun_out/${tag}_ncu_bench.log 2>&1; echo "launches rc=$?"
NF="ncu --set full --clock-control none --import-source on"
timeout 900 $NF -k regex:dawn_persistent -s 2 -c 1 -o gpurun_out/${tag}_c2 -f python tools/round_profile.py --solves 3 > gpurun_out/${tag}_ncu_c2.log 2>&1; echo "c2 rc=$?"
timeout 900 $NF -k regex:dawn_worklist -s 2 -c 1 -o gpurun_out/${tag}_wl -f python tools/round_profile.py --solves 3 > gpurun_out/${tag}_ncu_wl.log 2>&1; echo "wl rc=$?"
timeout 900 $NF -k regex:dawn_nearfar -s 0 -c 1 -o gpurun_out/${tag}_c4 -f python tools/nearfar_probe.py --grid 4096 --means 8 --caps 64 --solves 1 > gpurun_out/${tag}_ncu_c4.log 2>&1; echo "c4 rc=$?"
timeout 900 $NF -k regex:dawn_batch_persistent -s 3 -c 1 -o gpurun_out/${tag}_c3 -f python tools/apsp_probe.py --k 128 --single 2 > gpurun_out/${tag}_ncu_c3.log 2>&1; echo "c3 rc=$?"
python tools/traffic_stamp.py --rep gpurun_out/${tag}_c2.ncu-rep --rep gpurun_out/${tag}_wl.ncu-rep --key c2_async_fp32 \
  --out gpurun_out/traffic.json --capture "$tag: dawn_persistent + dawn_worklist, tools/round_profile.py (C2 async fp32)" > /dev/null; echo "stamp rc=$?"
for k in c2 wl c4 c3; do python tools/ncu_summary.py --rep gpurun_out/${tag}_$k.ncu-rep --out gpurun_out/${tag}_${k}_ncu.md --title "$tag $k" > /dev/null; done
python tools/ncu_summary.py --launches gpurun_out/${tag}_launches.csv --out gpurun_out/${tag}_launches.md --title "$tag launch list (bench.py --steps 3 --warmup 3)" > /dev/null

# reports are ~45 MB each (imported source): keep the summaries, raw pages and gzipped source pages
for k in c2 wl c4 c3; do
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page raw --csv > gpurun_out/${tag}_${k}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/${tag}_${k}_source.csv.gz
  mkdir -p /tmp/ncu_reps; mv gpurun_out/${tag}_$k.ncu-rep /tmp/ncu_reps/
done
du -sh gpurun_out
