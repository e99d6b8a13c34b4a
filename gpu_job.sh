timeout 900 python -m pytest tests/test_gpu_layer.py -x -q -p no:cacheprovider 2>&1 | tail -5
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
