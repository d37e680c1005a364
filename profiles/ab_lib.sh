set -e
F="--steps 5 --warmup 3 --no-cpu --no-e2e --no-onpolicy --no-recompute --no-ref-diag --no-dropin"
for r in 1 2 3; do
  for L in new prev; do
    if [ $L = new ]; then python bench.py $F > gpurun_out/ab_$L$r.json 2>/dev/null; else ICEPOP_B200_LIB=build/prev.so python bench.py $F > gpurun_out/ab_$L$r.json 2>/dev/null; fi
    python -c "
import json;d=json.loads(open('gpurun_out/ab_$L$r.json').read().strip().splitlines()[-1]); k=d['kernels_ms']; print('$L', $r, d['value'], d['clocks']['sm_mhz'], 'K4', k['K4_dhidden'], 'K5', k['K5_dweight'], 'prep', k['bwd_prep'])"
  done
done
