python tools/gemm_bench.py --env MOE_STORE_HINT --variants 0,1 --rounds 3
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-decode"
for h in 0 1; do MOE_STORE_HINT=$h $CMD > gpurun_out/plain.log 2>&1 && MOE_STORE_HINT=$h ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm_bf16" --csv --log-file gpurun_out/hint$h.csv $CMD > gpurun_out/ncu_launch.log 2>&1; done
