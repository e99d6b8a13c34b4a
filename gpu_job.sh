timeout 300 python -m pytest tests/test_gpu_layer.py -x -q -p no:cacheprovider -k "config3 or golden or fused" 2>&1 | tail -2
for r in 1 2; do for p in 0 1 2 3; do MOE_PREFETCH=$p python bench.py --steps 30 --no-decode --no-cpu-baseline > /tmp/b.json 2>/dev/null; python -c "
import json;d=json.load(open('/tmp/b.json'));ph=d['phases_ms'];print('pf=$p', round(d['ms_per_step'],3), {k:round(v,4) for k,v in ph.items()}, d['clocks']['sm_mhz'])"; done; done
