#!/usr/bin/env python
"""The paper's Section VI sweeps on the B200 engine, written as the
reference's benchmark CSV (bench.hpp:296-316: subject, backend, parameter,
value, mean_s, min_s, max_s, trials, budget_s, realtime -- the pinned header
of test_bench.cpp:148-151, in its number format) EXTENDED with percentile
and device columns the reference's TimingRecord (bench.hpp:61-74) lacks:

    p50_s, p99_s            host-timed process() latency percentiles
    device_p50_s, device_p99_s   device time of all of a block's work
    k_back_gbps             streaming kernel, algorithmic bytes / launch time

Semantics follow bench::run_sweep (bench.hpp:177-260) and SweepSpec's
defaults (bench.hpp:44-59): one input, broadcast synthesis; defaults 48 kHz,
block 128, 32 channels, 10 s synthesis, 1 s canceller; a swept parameter
overrides one default; filters N(0,1)/sqrt(n); `trials` single-block calls
after `warmup` calls, steady_clock around each; realtime = mean < budget.

    python tools/sweep_csv.py --subject auralizer --parameter block_size \
        --values 32,64,128,256,512,1024 --trials 2000 -o profiles/sweep.csv
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_04390_b200 as A  # noqa: E402

HEADER = "subject,backend,parameter,value,mean_s,min_s,max_s,trials,budget_s,realtime"
EXTRA = "p50_s,p99_s,device_p50_s,device_p99_s,k_back_gbps"
DEFAULTS = dict(sample_rate_hz=48000, block_size=128, channels=32, synth_length_s=10.0,
                fc_length_s=1.0)
PAPER_VALUES = {  # bench.hpp default_sweep_values
    "block_size": [16, 32, 64, 128, 256, 512, 1024, 2048, 4096],
    "channels": [1, 2, 4, 8, 16, 32, 64, 128],
    "filter_length_s": [0.5, 1, 2, 4, 8, 10, 16, 20],
    "fc_length_s": [0.1, 0.25, 0.5, 1, 2, 5],
}


def fmt(x):
    """Shortest round-trippable decimal, as the reference's format_double."""
    if isinstance(x, int) or float(x).is_integer() and abs(x) < 1e15:
        return str(int(x))
    return repr(float(x))


def resolve(parameter, value):
    """bench.hpp detail::resolve: the swept parameter overrides one default
    (filter_length_s is the synthesis length)."""
    r = dict(DEFAULTS)
    r["synth_length_s" if parameter == "filter_length_s" else parameter] = value
    fs = r["sample_rate_hz"]
    return (int(r["block_size"]), int(r["channels"]), int(round(r["synth_length_s"] * fs)),
            int(round(r["fc_length_s"] * fs)), fs)


def run(subject, parameter, values, trials, warmup, seed):
    rows = []
    for i, v in enumerate(values):
        N, C, n_h, n_hf, fs = resolve(parameter, v)
        rng = np.random.default_rng(seed + i)
        synth = [rng.standard_normal(n_h, dtype=np.float32) / np.float32(np.sqrt(n_h)) for _ in range(C)]
        cfg = A.make_config(fs, N, 1, C)
        try:
            if subject == "convolver":
                e = A.Convolver(synth, cfg)
            else:
                fc = [rng.standard_normal(n_hf, dtype=np.float32) / np.float32(np.sqrt(n_hf)) * 0.1
                      for _ in range(C)]
                e = A.Auralizer(synth, fc, cfg)
        except A.Error as err:
            if err.code == A.ErrorCode.out_of_memory:
                print(f"sweep: skipping {parameter}={v}: out of memory", file=sys.stderr)
                continue
            raise
        pool = rng.standard_normal((min(trials, 64), 1, N)).astype(np.float32)
        e.time_host_blocks(pool, warmup)
        host = e.time_host_blocks(pool, trials).astype(np.float64) * 1e-6
        _, dev = e.time_device_blocks(min(trials, 2000), pool)
        dev = dev.astype(np.float64) * 1e-6
        gbps = None
        ph = e.profile_phases(3)
        if ph.get("k_back", (0, 0))[1] > 0:
            us = e.time_phase("k_back", 10)
            gbps = ph["k_back"][1] / (us * 1e-6) / 1e9
        budget = N / fs
        mean = float(host.mean())
        rows.append([subject, "accelerator", parameter, v, mean, float(host.min()), float(host.max()), trials,
                     budget, "true" if mean < budget else "false", float(np.percentile(host, 50)),
                     float(np.percentile(host, 99)), float(np.percentile(dev, 50)), float(np.percentile(dev, 99)),
                     gbps if gbps is not None else ""])
        e.close()
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--subject", default="convolver", choices=["convolver", "auralizer"])
    ap.add_argument("--parameter", default="block_size", choices=sorted(PAPER_VALUES))
    ap.add_argument("--values", default=None, help="comma-separated; default: the reference's sweep")
    ap.add_argument("--trials", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("-o", "--out", default="-")
    args = ap.parse_args()
    values = ([float(x) for x in args.values.split(",")] if args.values else PAPER_VALUES[args.parameter])
    values = [int(x) if float(x).is_integer() and args.parameter in ("block_size", "channels") else x
              for x in values]
    rows = run(args.subject, args.parameter, values, args.trials, args.warmup, args.seed)
    lines = [HEADER + "," + EXTRA] + [",".join(fmt(x) if not isinstance(x, str) else x for x in r) for r in rows]
    text = "\n".join(lines) + "\n"
    if args.out == "-":
        sys.stdout.write(text)
    else:
        with open(args.out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
