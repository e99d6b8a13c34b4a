for i in 1 2 3; do
for cfg in "MOE_COMBINE_COAL=0 MOE_COMBINE_BN512=0" "MOE_COMBINE_COAL=1 MOE_COMBINE_BN512=0" "MOE_COMBINE_COAL=1 MOE_COMBINE_BN512=1"; do
  env $cfg python bench.py --steps 20 --warmup 5 --no-decode --train-steps 0 --no-cpu-baseline --sustained-s 2 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['sustained']
print('$cfg', 'burst', round(d['value']/1e6,3), 'M', {k: round(x,4) for k,x in d['phases_ms'].items() if k.startswith('gemm')}, 'sustained', round(s['tokens_per_s']/1e6,3), 'M', round(s['gemm_ms'],4), s['clocks'] and s['clocks']['sm_mhz'])"
done; done
