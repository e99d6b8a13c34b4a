# interleaved A/B of two builds of the library on a workload (burst + sustained)
# usage: bash tools/ab_lib.sh WORKLOAD "libA.so libB.so" [rounds]
W=$1; LIBS=$2; R=${3:-3}
for i in $(seq 1 $R); do for l in $LIBS; do
  MOE_B200_LIB=$l python bench.py --workload $W --steps 20 --warmup 5 --no-decode --train-steps 0 --no-cpu-baseline --sustained-s 2 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['sustained']
print('$W', '$(basename $l)', 'burst', round(d['value']/1e6,3), 'M', {k: round(x,4) for k,x in d['phases_ms'].items()}, 'sustained', round(s['tokens_per_s']/1e6,3), 'M gemm', round(s['gemm_ms'],4), s['clocks'] and s['clocks']['sm_mhz'])"
done; done
