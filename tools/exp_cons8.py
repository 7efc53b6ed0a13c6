"""Experiment (GPU box): the constrained update at c3 with the eight-points-
per-thread kernel (k_afc_constrain8) against the one-warp-per-unit kernel:
bit-identity of y, f^ and W over 30 blocks, and the block timeline."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2509_04390_b200 as A
from conftest import decaying_filters
N, L = 64, 64
rng = np.random.default_rng(0)
synth = decaying_filters(rng, L, 480000)
fc = decaying_filters(rng, L, 48000, t60_s=0.3, scale=0.1)
cfg = A.make_config(48000, N, 1, L)
mics = rng.standard_normal((30, 1, N)).astype(np.float32)
runs = {}
CASES = [json.loads(c) for c in sys.argv[1:]] or [{"AURA_B200_CONS_OCT": "1"}]
for env in CASES + [{"AURA_B200_CONS_OCT": "0"}]:
    for k in [k for k in os.environ if k.startswith("AURA_B200_")]:
        os.environ.pop(k, None)
    os.environ.update(env)
    e = A.Auralizer(list(synth), list(fc), cfg, afc=A.AfcParams(0.005, 0.9, None, True))
    ys = np.stack([e.process(m).copy() for m in mics])
    key = json.dumps(env)
    runs[key] = (ys, e.feedback_estimate().copy(), e.coeffs().copy())
    e.time_device_blocks(20, mics)
    span = e.time_device_span(200, mics)
    tr = e.trace_blocks(16)
    print(json.dumps({"env": env, "span_us": round(span, 2),
                      "timeline": {k: [round(float(np.median(v[:, 0])), 2), round(float(np.median(v[:, 1])), 2)]
                                   for k, v in tr.items() if k in ("k_afc_constrain", "k_back", "k_reduce", "cycle")}}),
          flush=True)
    e.close()
ref = runs[json.dumps({"AURA_B200_CONS_OCT": "0"})]
for k, v in runs.items():
    print(k, "bit-identical to the one-warp kernel:",
          all(np.array_equal(x, y) for x, y in zip(v, ref)), flush=True)
