timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q -p no:cacheprovider 2>&1 | tail -2
python tools/gemm_bench.py --env MOE_STORE_HINT --variants 1 --rounds 3
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2>gpurun_out/bench.err; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['phases_ms'],d['clocks'])"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-decode"
ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16_tc_kernel" -s 1 -c 2 -o gpurun_out/r1e_full $CMD > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
