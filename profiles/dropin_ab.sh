F="--steps 3 --warmup 3 --no-cpu --no-e2e --no-onpolicy --no-recompute --no-ref-diag --no-kernel-timing"
for r in 1 2; do
for L in new prev; do
  if [ $L = new ]; then python bench.py $F > gpurun_out/dab_$L.json 2>/dev/null; else ICEPOP_B200_LIB=build/prev.so python bench.py $F > gpurun_out/dab_$L.json 2>/dev/null; fi
  python -c "
import json;d=json.loads(open('gpurun_out/dab_$L.json').read().strip().splitlines()[-1]); print('$L', d['value'], d['dropin_c1']['fresh_grad'], d['dropin_c1']['grad_out'])"
done; done
