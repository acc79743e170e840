# usage: bash tools/gpurun_iter.sh TAG [configs] -- GPU tests (stop at first failure), bench lines and launch lists
TAG=${1:-it}; CONFIGS=${2:-"c2 c3 c4"}
O=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
tail -3 $O/${TAG}_pytest.log
timeout 300 python tools/phase_prof.py c3 > $O/${TAG}_phase_c3.txt 2>&1
for c in $CONFIGS; do timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; done
for c in $CONFIGS; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:enc_|sif_(parse|dcrc|scatter|dfinal|dec_small)' -c 40 --csv --log-file $O/${TAG}_launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
