set -x
for c in c2 c3 c4; do timeout 300 python tools/phase_prof.py $c > gpurun_out/r1_phase_$c.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'sif_(encode|parse|scatter)' -c 12 --csv --log-file gpurun_out/r1_launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1_ncu_launch.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sif_encode_kernel -s 3 -c 1 -o gpurun_out/r1_enc_c3 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1_ncu_enc3.log 2>&1
