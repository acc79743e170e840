# usage: bash tools/gpurun_quick.sh TAG  -- GPU tests, 1-GPU bench of c2/c3/c4, launch list for c2
TAG=${1:-q}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'enc_|sif_(parse|scatter)' -c 40 --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'enc_|sif_(parse|scatter)' -c 40 --csv --log-file gpurun_out/${TAG}_launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'enc_|sif_(parse|scatter)' -c 40 --csv --log-file gpurun_out/${TAG}_launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
