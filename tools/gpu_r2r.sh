#!/bin/bash
O=gpurun_out/r2r
mkdir -p $O
timeout 1200 python tools/exp_knobs.py c3 '{}' '{"AURA_B200_LATE_AT": 0.5}' '{"AURA_B200_LATE_AT": 0.7}' '{"AURA_B200_LATE_AT": 0.9}' '{}' '{"AURA_B200_LATE_AT": 0.5}' > $O/knobs.jsonl 2> $O/knobs.err
timeout 900 python tools/exp_knobs.py c5 '{}' '{"AURA_B200_LATE_AT": 0.5}' >> $O/knobs.jsonl 2>> $O/knobs.err
timeout 900 python tools/exp_knobs.py c4 '{}' '{"AURA_B200_LATE_AT": 0.5}' >> $O/knobs.jsonl 2>> $O/knobs.err
python3 - <<'PY'
import json
for l in open('gpurun_out/r2r/knobs.jsonl'):
    d=json.loads(l); t=d['trace']
    print(d['env'], 'span', round(d['span_mean_us'],2), 'ev', round(d['events_p50'],2), round(d['events_p99'],2), 'e2e', round(d['e2e_p50'],2), round(d['e2e_p99'],2), 'back', t.get('k_back'), 'red', t.get('k_reduce'), 'cyc', t.get('cycle'))
PY
tail -3 $O/knobs.err
