#!/bin/bash
O=gpurun_out/r2s
mkdir -p $O
timeout 1500 python tools/exp_knobs.py c3 '{}' '{"AURA_B200_H_L2_MB": 20}' '{"AURA_B200_H_L2_MB": 40}' '{"AURA_B200_H_L2_MB": 60}' '{"AURA_B200_H_L2_MB": 80}' '{"AURA_B200_W_L2_MB": 200}' '{"AURA_B200_W_L2_MB": 200, "AURA_B200_H_L2_MB": 40}' '{}' > $O/knobs.jsonl 2> $O/knobs.err
python3 - <<'PY'
import json
for l in open('gpurun_out/r2s/knobs.jsonl'):
    d=json.loads(l); t=d['trace']
    print(d['env'], 'span', round(d['span_mean_us'],2), 'ev', round(d['events_p50'],2), round(d['events_p99'],2), 'e2e', round(d['e2e_p50'],2), round(d['e2e_p99'],2), 'back', t.get('k_back'), 'red', t.get('k_reduce'), 'cyc', t.get('cycle'))
PY
tail -3 $O/knobs.err
