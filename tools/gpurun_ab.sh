# usage: bash tools/gpurun_ab.sh TAG -- GPU tests, then per-kernel times of C2 and C4 (tools/kprof.py) and their bench lines
O=gpurun_out; TAG=${1:-ab}
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 300 python tools/kprof.py 0 1024 196 256 fp32 > $O/${TAG}_kp_c2.txt 2>&1
timeout 300 python tools/kprof.py 1 2048 4096 32 bf16 > $O/${TAG}_kp_c4.txt 2>&1
for c in c2 c4; do timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; done
