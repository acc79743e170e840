# usage: bash tools/gpurun_lam3.sh TAG -- GPU tests, C2 / C4 (lambda 0 and 0.1) per-kernel times, C2 line, C4 sweep
O=gpurun_out; TAG=${1:-lam3}
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 300 python tools/kprof.py 1 2048 4096 32 bf16 lam=0.1 > $O/${TAG}_kp_c4_lam0.1.txt 2>&1
timeout 300 python tools/kprof.py 1 2048 4096 32 bf16 > $O/${TAG}_kp_c4.txt 2>&1
timeout 300 python tools/kprof.py 0 1024 196 256 fp32 > $O/${TAG}_kp_c2.txt 2>&1
timeout 400 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > $O/${TAG}_bench_c2.json 2> $O/${TAG}_bench_c2.err
timeout 900 python bench.py --config c4sweep --steps 3 --warmup 3 --no-cpu-baseline > $O/${TAG}_bench_c4sweep.json 2> $O/${TAG}_bench_c4sweep.err
