O=gpurun_out; TAG=${1:-lam}
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
for lam in 0.0 0.1; do timeout 300 python tools/kprof.py 1 2048 4096 32 bf16 lam=$lam > $O/${TAG}_kp_c4_lam$lam.txt 2>&1; done
timeout 300 python tools/kprof.py 0 1024 196 256 fp32 lam=0.1 > $O/${TAG}_kp_c2_lam0.1.txt 2>&1
timeout 900 python bench.py --config c4sweep --steps 3 --warmup 3 --no-cpu-baseline > $O/${TAG}_bench_c4sweep.json 2> $O/${TAG}_bench_c4sweep.err
