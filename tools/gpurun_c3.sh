O=gpurun_out; TAG=${1:-c3}
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 400 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $O/${TAG}_bench_c3.json 2> $O/${TAG}_bench_c3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:enc_token|sif_dec_small' -c 20 --csv --log-file $O/${TAG}_launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
