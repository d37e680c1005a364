# C1 A/B of library builds (in-tree "tree" + build/<name>.so in $LIBS), R rounds, kernel timings
set -e
R=${R:-2}
F="--config c1 --steps 20 --warmup 5 --no-cpu --no-e2e --no-dropin --no-ref-diag"
for r in $(seq 1 $R); do
  for L in tree $LIBS; do
    if [ $L = tree ]; then python bench.py $F > gpurun_out/c1_$L$r.json 2>/dev/null; else ICEPOP_B200_LIB=build/$L.so python bench.py $F > gpurun_out/c1_$L$r.json 2>/dev/null; fi
    python -c "
import json;d=json.loads(open('gpurun_out/c1_$L$r.json').read().strip().splitlines()[-1]); k=d['kernels_ms']; rc=d['recompute']
print('%-9s' % '$L', $r, 'step', d['ms_per_step'], 'K1', k['K1_fwd_lse'], 'prep', k['bwd_prep'], 'K4', k['K4_dhidden'], 'K5', k['K5_dweight'], '| rc step', rc['ms_per_step'], 'K3', rc['kernels_ms']['K3_dz'], 'onp', d['on_policy']['ms_per_step'])"
  done
done
