timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q -p no:cacheprovider 2>&1 | tail -3
MOE_GEMM_VARIANT=1 timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q -p no:cacheprovider 2>&1 | tail -2
python tools/gemm_bench.py --rounds 3
