# usage: bash tools/gpurun_bench.sh TAG -- GPU tests + smoke + 1-GPU bench lines of c2/c3/c4 (+ reference arm)
TAG=${1:-r1}
O=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
for c in c2 c3 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_ref_c2.json 2> $O/${TAG}_bench_ref_c2.err
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --depth 2 > $O/${TAG}_bench_c5.json 2> $O/${TAG}_bench_c5.err
timeout 300 python bench.py --impl reference --config c5 --steps 2 --warmup 1 > $O/${TAG}_bench_ref_c5.json 2> $O/${TAG}_bench_ref_c5.err
