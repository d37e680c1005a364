# Interleaved A/B of environment knobs on one box (headline + kernel timings), R rounds.
# usage: KNOBS="BASE=1 ICEPOP_EPI_SLEEP_NS=200" R=3 bash profiles/knob_ab.sh
set -e
F=${F:-"--steps 5 --warmup 3 --no-cpu --no-e2e --no-onpolicy --no-recompute --no-ref-diag --no-dropin"}
R=${R:-3}
for r in $(seq 1 $R); do
  for kv in $KNOBS; do
    env $kv python bench.py $F > gpurun_out/knob.json 2>/dev/null
    python -c "
import json;d=json.loads(open('gpurun_out/knob.json').read().strip().splitlines()[-1]); k=d['kernels_ms']
print('%-26s' % '$kv', $r, d['value'], d['clocks']['sm_mhz'], 'K1', k.get('K1_fwd_lse'), 'K4', k['K4_dhidden'], 'K5', k['K5_dweight'])"
  done
done
