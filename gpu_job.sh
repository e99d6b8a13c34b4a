timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q -p no:cacheprovider 2>&1 | tail -2
python tools/gemm_bench.py --rounds 2 --variants 0
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm_bf16|scatter_kernel|combine_kernel|plan_scan" --csv --log-file gpurun_out/r1b_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
