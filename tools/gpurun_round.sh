set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r1_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1
for c in c2 c3 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r1_bench_$c.json 2> gpurun_out/r1_bench_$c.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r1_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sif_encode_kernel -s 3 -c 1 -o gpurun_out/r1_enc_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1_ncu_enc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sif_scatter_kernel -s 3 -c 1 -o gpurun_out/r1_dec_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1_ncu_dec.log 2>&1
ls -la gpurun_out
