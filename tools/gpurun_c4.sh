O=gpurun_out; TAG=${1:-c4}
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 300 python tools/kprof.py 1 2048 4096 32 bf16 > $O/${TAG}_kp_c4.txt 2>&1
timeout 400 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > $O/${TAG}_bench_c4.json 2> $O/${TAG}_bench_c4.err
timeout 400 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $O/${TAG}_bench_c3.json 2> $O/${TAG}_bench_c3.err
