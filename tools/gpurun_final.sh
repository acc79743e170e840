# usage: bash tools/gpurun_final.sh TAG -- round evidence on one B200: GPU tests, smoke, bench lines of every
# config (CPU baseline on), reference arms, launch lists and ncu --set full summaries (profiles/TAG_*_ncu.txt)
TAG=${1:-r2z}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,driver_version --format=csv > $O/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
# C1 (host-latency bound) first, before the CPU-baseline pools of the other lines, 100 steps
timeout 300 python bench.py --config c1 --steps 100 --warmup 10 > $O/${TAG}_bench_c1.json 2> $O/${TAG}_bench_c1.err
for c in c2 c3 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; done
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > $O/${TAG}_bench_c5.json 2> $O/${TAG}_bench_c5.err
timeout 900 python bench.py --config c4sweep --steps 3 --warmup 3 > $O/${TAG}_bench_c4sweep.json 2> $O/${TAG}_bench_c4sweep.err
for c in c2 c3 c5; do timeout 600 python bench.py --impl reference --config $c --steps 2 --warmup 1 > $O/${TAG}_bench_ref_$c.json 2> $O/${TAG}_bench_ref_$c.err; done
KRE='regex:enc_|sif_(parse|dcrc|scatter|dfinal|dec_small)'
for ck in c2:13 c3:2 c4:17; do
  c=${ck%%:*}; K=${ck##*:}
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c $((3 * K)) --csv --log-file $O/${TAG}_launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k "$KRE" -s $K -c $K -o $O/${TAG}_full_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --depth 1 > /dev/null 2>&1
done
python tools/make_profiles.py ${TAG} c2:$O/${TAG}_full_c2.ncu-rep c3:$O/${TAG}_full_c3.ncu-rep c4:$O/${TAG}_full_c4.ncu-rep > $O/${TAG}_profiles.log 2>&1
mkdir -p $O/profiles && cp profiles/${TAG}_*_ncu.txt profiles/ncu_traffic.json $O/profiles/ 2>/dev/null
rm -f $O/${TAG}_full_c3.ncu-rep $O/${TAG}_full_c4.ncu-rep
du -sh $O
