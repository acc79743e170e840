for sw in 1024 1280 1536 2048; do
 SIF_SEGW=$sw timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('segw $sw', d['value'], d['ms_per_step'], d['kernels']['sif_scatter_kernel']['us_per_launch'])" >> gpurun_out/segw.txt
done
