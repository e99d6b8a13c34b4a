# interleaved A/B of an environment knob on a workload (burst, L2-flushed steps)
# usage: bash tools/ab_wl.sh WORKLOAD VAR "v0 v1" [rounds]
W=$1; VAR=$2; VALS=$3; R=${4:-2}
for i in $(seq 1 $R); do for v in $VALS; do
  env $VAR=$v python bench.py --workload $W --steps 50 --warmup 5 --no-decode --train-steps 0 --no-cpu-baseline --sustained-s 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['sustained']
print('$W $VAR=$v', round(d['value']/1e6,3), 'M', {k: round(x,4) for k,x in d['phases_ms'].items()}, 'sustained', round(s['tokens_per_s']/1e6,3))"
done; done
