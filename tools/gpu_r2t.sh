#!/bin/bash
O=gpurun_out/r2t
mkdir -p $O
timeout 1200 python tools/exp_knobs.py c3 '{}' '{"AURA_B200_AFC_TAIL": 1}' '{}' '{"AURA_B200_AFC_TAIL": 1}' > $O/knobs.jsonl 2> $O/knobs.err
timeout 600 python tools/exp_knobs.py c4 '{}' '{"AURA_B200_AFC_TAIL": 1}' >> $O/knobs.jsonl 2>> $O/knobs.err
python3 - <<'PY'
import json
for l in open('gpurun_out/r2t/knobs.jsonl'):
    d=json.loads(l); t=d['trace']
    print(d['env'], 'span', round(d['span_mean_us'],2), 'ev', round(d['events_p50'],2), round(d['events_p99'],2), 'e2e', round(d['e2e_p50'],2), round(d['e2e_p99'],2), 'back', t.get('k_back'), 'red', t.get('k_reduce'), 'summed', t.get('afc_summed'), 'done', t.get('afc_done'), 'cyc', t.get('cycle'))
PY
tail -3 $O/knobs.err
