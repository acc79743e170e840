timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/q32_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q32_pytest.log
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/q32_bench_$c.json 2> gpurun_out/q32_bench_$c.err; done
python tools/phase_prof.py c3 > gpurun_out/q32_ph_c3.txt 2>&1
