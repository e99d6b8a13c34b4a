python tools/gemm_bench.py --env MOE_RASTER --variants 0,1 --rounds 4
