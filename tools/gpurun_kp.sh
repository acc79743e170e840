for lam in 0.0 0.1; do timeout 300 python tools/kprof.py 1 2048 4096 32 bf16 lam=$lam > gpurun_out/kp_c4_lam$lam.txt 2>&1; done
timeout 300 python tools/kprof.py 0 1024 196 256 fp32 lam=0.1 > gpurun_out/kp_c2_lam0.1.txt 2>&1
