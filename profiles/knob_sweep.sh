#!/bin/bash
# Interleaved A/B of the scheduling knobs on one box: each setting is a fresh process (the
# switches are read once per process); two rounds so that box drift shows.
set -u
out=${1:-gpurun_out/knob_sweep.jsonl}
: > "$out"
for round in 1 2; do
  for kv in "BASE=1" "ICEPOP_K1_WIDE=1" "ICEPOP_GROUP_M=8" "ICEPOP_GROUP_M=24" "ICEPOP_GROUP_M_LONG=4" \
            "ICEPOP_SYNC_KB=32" "ICEPOP_SYNC_KB=128"; do
    env "$kv" python bench.py --steps 4 --warmup 2 --no-cpu --no-e2e --no-onpolicy --no-recompute --no-ref-diag \
        --no-dropin --no-kernel-timing 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({'knob':'$kv','round':$round,'value':d['value'],'ms':d['ms_per_step'],'mhz':(d.get('clocks') or {}).get('sm_mhz')}))" >> "$out"
  done
done
cat "$out"
