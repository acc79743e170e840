# usage: bash tools/gpurun_r2.sh TAG -- GPU tests, smoke, 1-GPU bench c1..c5 (+reference c2), launch lists c2/c3/c4
TAG=${1:-r2}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
for c in c2 c3 c4 c5 c1; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_ref_c2.json 2> $O/${TAG}_bench_ref_c2.err
KRE='regex:enc_|sif_(parse|dcrc|scatter|dfinal)'
for c in c2 c3 c4; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 60 --csv --log-file $O/${TAG}_launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
