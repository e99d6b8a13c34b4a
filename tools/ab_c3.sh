# interleaved A/B of an environment knob on the C3 step (burst + 2 s sustained)
# usage: bash tools/ab_c3.sh VAR "v0 v1" [rounds]
VAR=$1; VALS=$2; R=${3:-2}
for i in $(seq 1 $R); do for v in $VALS; do
  env $VAR=$v python bench.py --steps 20 --warmup 5 --no-decode --train-steps 0 --no-cpu-baseline --sustained-s 2 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['sustained']
print('$VAR=$v', 'burst', round(d['value']/1e6,3), 'M', {k: round(x,4) for k,x in d['phases_ms'].items() if k.startswith('gemm')}, 'sustained', round(s['tokens_per_s']/1e6,3), 'M', round(s['gemm_ms'],4), s['clocks'] and s['clocks']['sm_mhz'])"
done; done
