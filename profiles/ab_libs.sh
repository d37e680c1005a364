# A/B/... of library builds on one box: the in-tree one ("tree") and each build/<name>.so given
# in $LIBS, interleaved, R rounds; bench flags in $F (default: headline + kernel timings).
set -e
F=${F:-"--steps 5 --warmup 3 --no-cpu --no-e2e --no-onpolicy --no-recompute --no-ref-diag --no-dropin"}
R=${R:-3}
for r in $(seq 1 $R); do
  for L in tree $LIBS; do
    if [ $L = tree ]; then python bench.py $F > gpurun_out/abl_$L$r.json 2>/dev/null; else ICEPOP_B200_LIB=build/$L.so python bench.py $F > gpurun_out/abl_$L$r.json 2>/dev/null; fi
    python -c "
import json;d=json.loads(open('gpurun_out/abl_$L$r.json').read().strip().splitlines()[-1]); k=d['kernels_ms']
print('%-10s' % '$L', $r, d['value'], d['clocks']['sm_mhz'], 'K1', k.get('K1_fwd_lse'), 'K4', k['K4_dhidden'], 'K5', k['K5_dweight'])"
  done
done
