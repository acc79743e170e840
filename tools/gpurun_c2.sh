# usage: bash tools/gpurun_c2.sh TAG -- GPU tests (optional SKIP_TESTS=1), c2 bench + c2 launch list
TAG=${1:-q}
[ -z "$SKIP_TESTS" ] && { timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log; }
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'enc_|sif_(parse|scatter)' -c 40 --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
