# A/B of two builds of the library on one box: the in-tree one ("new") and build/prev.so
# ("prev"), alternating, R rounds; bench flags in $F (default: headline only).
set -e
F=${F:-"--steps 5 --warmup 3 --no-cpu --no-e2e --no-onpolicy --no-recompute --no-ref-diag --no-dropin"}
R=${R:-3}
for r in $(seq 1 $R); do
  for L in new prev; do
    if [ $L = new ]; then python bench.py $F > gpurun_out/ab_$L$r.json 2>/dev/null; else ICEPOP_B200_LIB=build/prev.so python bench.py $F > gpurun_out/ab_$L$r.json 2>/dev/null; fi
    python -c "
import json;d=json.loads(open('gpurun_out/ab_$L$r.json').read().strip().splitlines()[-1]); k=d['kernels_ms']
rc=d.get('recompute',{}).get('value'); op=d.get('on_policy',{}).get('value')
print('$L', $r, d['value'], d['clocks']['sm_mhz'], 'recompute', rc, 'on_policy', op, 'K4', k['K4_dhidden'], 'K5', k['K5_dweight'])"
  done
done
