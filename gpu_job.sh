python tools/gate_bench.py
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_routing.py -x -q -p no:cacheprovider 2>&1 | tail -2
