#!/usr/bin/env python
"""Benchmark of the B200 UPOLS + feedback-canceller block loop.

Metric (BASELINE.json): per-block latency p50/p99 (us) and maximum
real-time channels x taps at 48 kHz. One "step" = one audio block through
the whole path (m~ = g m - f^, r2c, FDL MAC over all partitions x
loudspeakers, c2r + overlap-save, canceller r2c, canceller MAC with the NLMS
update, f^ for the next block).

    python bench.py [--config c3] [--gpus N] [--steps K] [--warmup W]
    python bench.py --impl reference ...   # the reference's CPU path

value  = p99 device time per block, inputs resident in HBM, CUDA events on
         the engine stream (lower is better).
e2e    = p99 of aura_b200_process() with host buffers (host->device input,
         all kernels, device->host output, completion wait), steady_clock.
max_realtime = the metric's second half: the largest loudspeaker count at
         the config's taps whose block p99 fits N/f_s on the device AND whose
         process() calls, paced on the real-time grid, return within N/f_s
         (time-boxed binary search; per GPU, summed over GPUs at N > 1).
c5     = BASELINE configs[4] (1 x 512, 96 kHz, 20 s), the loudspeakers split
         over the N GPUs (strong scaling), reported beside the headline.

--gpus N without torchrun re-launches itself under torch.distributed.run
(one process per GPU); every number is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("per-block latency p50/p99 (µs) and max real-time channels×taps "
          "at 48 kHz")

# BASELINE.json configs (SURVEY 8(d) sizes); AFC length 1 s where on.
CONFIGS = {
    "c1": dict(fs=48000, N=256, Q=1, L=2, n_h=96000, afc=False,
               desc="c1: 1 input x 2 loudspeakers, 48 kHz, block 256, 2 s IR (96k taps), no AFC"),
    "c2": dict(fs=48000, N=128, Q=1, L=16, n_h=480000, afc=False,
               desc="c2: 1 input x 16 loudspeakers, 48 kHz, block 128, 10 s IR (480k taps)"),
    "c3": dict(fs=48000, N=64, Q=1, L=64, n_h=480000, afc=True, n_hf=48000, mu=0.005,
               desc="c3: 1 input x 64 loudspeakers, 48 kHz, block 64, 10 s IR (480k taps), "
                    "PBFDAF feedback canceller 1 s (48k taps) with NLMS update",
               ref_desc="c3: 1 input x 64 loudspeakers, 48 kHz, block 64, 10 s IR (480k taps), "
                        "feedback canceller 1 s (48k taps) with a FIXED F^ (the reference has no "
                        "NLMS; same MAC bytes minus the W write)"),
    "c4": dict(fs=48000, N=64, Q=4, L=64, n_h=576000, afc=True, n_hf=48000, mu=0.005,
               desc="c4: 4 inputs x 64 loudspeakers MIMO, 48 kHz, block 64, 12 s IR (576k taps), "
                    "AFC 1 s with NLMS",
               ref_desc="c4: 4 inputs x 64 loudspeakers (4 reference Auralizers, the same MAC "
                        "work), 48 kHz, block 64, 12 s IR (576k taps), FIXED-F^ canceller 1 s"),
    "c5": dict(fs=96000, N=128, Q=1, L=512, n_h=1920000, afc=False,
               desc="c5: 1 input x 512 loudspeakers, 96 kHz, block 128, 20 s IR (1.92M taps)"),
}


def decaying_noise(rng, rows, n, fs, t60_s=None, scale=1.0):
    """Exponentially decaying noise IRs: n(t) 10^(-3 t / T60), sum h^2 = 1
    (SURVEY 8(d)); T60 = IR length unless given."""
    t60 = n / fs if t60_s is None else t60_s
    env = (10.0 ** (-3.0 * np.arange(n, dtype=np.float64) / (t60 * fs))).astype(np.float32)
    out = np.empty((rows, n), np.float32)
    for r in range(rows):
        h = rng.standard_normal(n, dtype=np.float32) * env
        h *= np.float32(scale / np.sqrt(np.dot(h.astype(np.float64), h)))
        out[r] = h
    return out


class LazyRows:
    """Row r of a decaying-noise filter set, generated on first use (seeded
    per row): a loudspeaker shard materialises only its own rows."""

    def __init__(self, n_rows, n_taps, fs, t60_s=None, scale=1.0, seed=1000):
        self.n_rows, self.n_taps, self.fs = n_rows, n_taps, fs
        self.t60_s, self.scale, self.seed = t60_s, scale, seed

    def __len__(self):
        return self.n_rows

    def __getitem__(self, r):
        if not 0 <= r < self.n_rows:
            raise IndexError(r)
        rng = np.random.default_rng((self.seed, r))
        return decaying_noise(rng, 1, self.n_taps, self.fs, self.t60_s, self.scale)[0]


def make_workload(cfg, seed=1000):
    rng = np.random.default_rng(seed)
    Q, L = cfg["Q"], cfg["L"]
    synth = decaying_noise(rng, Q * L, cfg["n_h"], cfg["fs"])
    fc = None
    if cfg["afc"]:
        fc = decaying_noise(rng, Q * L, cfg["n_hf"], cfg["fs"], t60_s=0.3, scale=0.1)
    mic = np.random.default_rng(7).standard_normal((64, Q, cfg["N"])).astype(np.float32)
    return synth, fc, mic


def pct(a, q):
    return float(np.percentile(np.asarray(a, np.float64), q))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(config_name, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f).get(config_name)
    except (OSError, ValueError):
        return None, None
    if not d or d.get("kernel") != kernel:
        return None, None
    return float(d["dram_read_bytes"] + d["dram_write_bytes"]), d.get("source")


READ_PROBE_GBS = 7379.1  # tools/bw_probe.cu on this pool's B200 (profiles/r1s3_c3_stream_kernel.md)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in getattr(self, "lines", []):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for name, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ reference arm

def reference_blocks(cfg, synth, fc, mic, blocks, warmup, backend="parallel", L_sub=None):
    """Time the UNMODIFIED reference (oracle/_ref: aura::Convolver /
    aura::Auralizer, ParallelBackend with hardware_concurrency workers) on the
    same synthetic inputs. Q > 1 (c4) is timed as Q single-input Auralizers
    (the same MAC work, Appendix B); the reference has no NLMS, so its
    canceller is the fixed-F^ one."""
    import oracle as O
    N, Q, L = cfg["N"], cfg["Q"], cfg["L"]
    if L_sub:
        L = L_sub
    t_setup = time.perf_counter()
    engines = []
    for q in range(Q):
        s = synth[q * cfg["L"]:q * cfg["L"] + L]
        if cfg["afc"]:
            f = fc[q * cfg["L"]:q * cfg["L"] + L]
            engines.append(O.RefAuralizer(s, f, N, L, backend=backend))
        else:
            engines.append(O.RefConvolver(s, N, 1, L, O.BROADCAST, backend=backend))
    t_setup = time.perf_counter() - t_setup
    times = []
    for b in range(warmup + blocks):
        m = mic[b % mic.shape[0]]
        t0 = time.perf_counter()
        for q, e in enumerate(engines):
            e.process(m[q:q + 1])
        t1 = time.perf_counter()
        if b >= warmup:
            times.append((t1 - t0) * 1e6)
    workers = O.ref_backend_workers(backend)
    return np.array(times), workers, t_setup


def cpu_sample_channels(cfg, max_taps=200e6):
    """Loudspeaker subset for the CPU reference when the full configuration's
    setup (make_partitioned_filters) would take minutes: (L_sub, scale) or
    (None, 1.0)."""
    taps = cfg["Q"] * cfg["L"] * cfg["n_h"]
    if taps <= max_taps:
        return None, 1.0
    L_sub = max(1, int(cfg["L"] * max_taps / taps))
    return L_sub, cfg["L"] / L_sub


def run_reference_arm(args, cfg, rank):
    if rank != 0:
        return 0
    cfg = sharded_cfg(cfg, int(os.environ.get("WORLD_SIZE", "1")), args.scaling)
    synth, fc, mic = make_workload(cfg)
    blocks = max(1, args.steps)
    L_sub, scale = cpu_sample_channels(cfg)
    us, workers, t_setup = reference_blocks(cfg, synth, fc, mic, blocks, args.warmup, L_sub=L_sub)
    us = us * scale
    p50, p99 = pct(us, 50), pct(us, 99)
    desc = cfg.get("ref_desc", cfg["desc"])
    sample = (f"{blocks} blocks of {desc} (after {args.warmup} warm-up), reference "
              f"ParallelBackend, -O3 -DNDEBUG -std=c++20; fixed-F^ canceller (the reference "
              f"has no NLMS); setup {t_setup:.1f} s excluded")
    if L_sub:
        sample += f"; {L_sub} of {cfg['L']} loudspeakers timed and scaled x{scale:.1f}"
    line = {
        "impl": "reference", "metric": METRIC, "value": p99, "unit": "us",
        "n_gpus": args.gpus, "steps": blocks, "warmup": args.warmup,
        "ms_per_step": float(np.mean(us)) / 1000.0, "higher_is_better": False,
        "scaling": args.scaling if args.gpus > 1 else "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": desc},
        "p50_us": p50, "p99_us": p99, "budget_us": 1e6 * cfg["N"] / cfg["fs"],
        "cpu_baseline": {"value": p99, "unit": "us", "cores": workers, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": p99, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- B200 arm

def make_engine(A, cfg, synth, fc, device=0, L=None, mu=None):
    N, Q = cfg["N"], cfg["Q"]
    L = cfg["L"] if L is None else L
    if L != cfg["L"]:
        idx = np.concatenate([np.arange(q * cfg["L"], q * cfg["L"] + L) for q in range(Q)])
        synth = synth[idx] if synth.shape[0] >= idx.max() + 1 else synth
        fc = fc[idx] if fc is not None else None
    backend = A.make_backend("gpu", device)
    ec = A.make_config(cfg["fs"], N, Q, L, mimo=Q > 1)
    if cfg["afc"]:
        m = cfg.get("mu", 0.0) if mu is None else mu
        return A.Auralizer(list(synth), list(fc), ec, backend,
                           afc=A.AfcParams(m, 0.9, None))
    mode = A.ChannelMode.mimo if Q > 1 else A.ChannelMode.broadcast
    return A.Convolver(list(synth), ec, mode, backend)


def aliased_rows(n_rows, n_taps, distinct=16, scale=1e-3, seed=3):
    """n_rows filter rows made of `distinct` random rows, aliased: timing does
    not depend on the filter values (the MAC streams every channel's spectra
    whatever they hold), and this keeps host setup cheap at L ~ 10^3."""
    rng = np.random.default_rng(seed)
    base = [rng.standard_normal(n_taps, dtype=np.float32) * np.float32(scale) for _ in range(distinct)]
    return [base[i % distinct] for i in range(n_rows)]


def max_realtime(A, cfg, device, blocks=300, budget_s=110.0):
    """The metric's second half (bench.hpp:245: real time = block time within
    N/f_s): the largest loudspeaker count L, taps fixed at the
    config's n_h, same canceller setting, for which BOTH
      - the device p99 of a block's whole work (front + background) < N/f_s,
      - the p99 latency of aura_b200_process() with host buffers, called on
        the real-time grid (one call every N/f_s), < N/f_s,
    binary search on L (resolution L/32), time-boxed to budget_s."""
    t_start = time.perf_counter()
    N, fs = cfg["N"], cfg["fs"]
    budget_us = 1e6 * N / fs
    Q = cfg["Q"]
    mic = np.random.default_rng(7).standard_normal((64, Q, N)).astype(np.float32)
    trials = []

    def fits(L):
        c = dict(cfg, L=L)
        synth = aliased_rows(Q * L, cfg["n_h"])
        fc = aliased_rows(Q * L, cfg["n_hf"], scale=1e-4, seed=4) if c["afc"] else None
        try:
            e = make_engine(A, c, synth, fc, device)
        except A.Error as err:
            if err.code == A.ErrorCode.out_of_memory:
                trials.append({"L": L, "fits": False, "why": "out of memory"})
                return False
            raise
        del synth, fc
        e.time_device_blocks(20, mic)
        _, us = e.time_device_blocks(blocks, mic)
        dev99 = pct(us, 99)
        host99 = None
        if dev99 < budget_us:
            e.time_host_blocks(mic, 20, pace_us=budget_us)
            host = e.time_host_blocks(mic, blocks, pace_us=budget_us)
            e.synchronize()
            host99 = pct(host, 99)
        e.close()
        ok = dev99 < budget_us and host99 is not None and host99 < budget_us
        trials.append({"L": L, "fits": ok, "device_p99_us": dev99, "paced_e2e_p99_us": host99})
        return ok

    lo, hi = cfg["L"], None
    if not fits(lo):
        return {"channels": 0, "trials": trials, "p99_criterion_us": budget_us}
    step = lo
    while hi is None and time.perf_counter() - t_start < budget_s:
        cand = lo + step
        if fits(cand):
            lo, step = cand, step * 2
        else:
            hi = cand
    while hi is not None and hi - lo > max(1, lo // 32) and time.perf_counter() - t_start < budget_s:
        mid = (lo + hi) // 2
        if fits(mid):
            lo = mid
        else:
            hi = mid
    return {"channels": lo, "taps": cfg["n_h"], "channels_x_taps": lo * cfg["n_h"],
            "upper_bound_channels": hi, "p99_criterion_us": budget_us,
            "criteria": "device block p99 AND paced process() e2e p99 < N/f_s",
            "search_s": time.perf_counter() - t_start, "trials": trials}


def l2_read_peak(footprint_bytes):
    """Measured L2-resident read bandwidth (GB/s) at this footprint:
    tools/bw_probe.cu BW_L2=1 on this pool's B200 (profiles/r2_l2_probe.jsonl;
    best of the LDG.128 and the cp.async.bulk stream, each a single launch
    re-reading a buffer of that size), interpolated in footprint."""
    path = os.path.join(ROOT, "profiles", "r2_l2_probe.jsonl")
    pts = {}
    try:
        with open(path) as f:
            for line in f:
                r = json.loads(line)
                if r.get("kind") in ("l2_ldg", "l2_bulk"):
                    mb = float(r["footprint_mb"])
                    pts[mb] = max(pts.get(mb, 0.0), float(r["GBps"]))
    except (OSError, ValueError):
        return None, None
    if not pts:
        return None, None
    xs = sorted(pts)
    mb = footprint_bytes / 1e6
    best = float(np.interp(mb, xs, [pts[x] for x in xs]))
    return best, "measured L2-resident read at %.0f MB (profiles/r2_l2_probe.jsonl)" % mb


L2_RESIDENT_BYTES = 80e6  # the engine's own rule (engine.cu plan_back: h_in_l2)


def roofline_regime(eng_bytes_footprint):
    """SURVEY 8(d)'s regime rule (footprint H + W + FDLs < L2/2 -> L2),
    with the engine's threshold: below 80 MB k_back streams the spectra with
    evict_normal hints and they stay in the 126 MB L2 between blocks (c2's
    65 MB included: warm ncu, profiles/r2_l2.md); above it, evict_first."""
    return "l2" if eng_bytes_footprint < L2_RESIDENT_BYTES else "hbm"


def c5_secondary(A, device, K, W, world=1, rank=0):
    """BASELINE configs[4] (1 x 512 loudspeakers, 96 kHz, N = 128, 20 s, no
    canceller) with its loudspeakers split over `world` GPUs (strong
    scaling: this rank runs its slice). Aliased filter rows (timing does not
    depend on values). Returns this rank's per-block device and e2e times."""
    from paper_2509_04390_b200 import shard as S
    c = CONFIGS["c5"]
    N, L = c["N"], c["L"]
    rows = aliased_rows(L, c["n_h"])
    ec = A.make_config(c["fs"], N, 1, L)
    t0 = time.perf_counter()
    conv = S.ShardedConvolver(rows, ec, world, rank, A.ChannelMode.broadcast, device)
    setup = time.perf_counter() - t0
    del rows
    mic = np.random.default_rng(7).standard_normal((64, 1, N)).astype(np.float32)
    e = conv.engine
    e.time_device_blocks(max(3, W), mic)
    _, dev = e.time_device_blocks(K, mic)
    host = e.time_host_blocks(mic, K)
    e.synchronize()
    out = {"dev": dev, "host": host, "channels": (conv.l0, conv.l1), "setup": setup,
           "bytes": e.profile_phases(3)["k_back"][1]}
    conv.close()
    return out


def c5_summary(parts, world):
    c = CONFIGS["c5"]
    dev = np.max(np.stack([p["dev"] for p in parts]), axis=0)
    host = np.max(np.stack([p["host"] for p in parts]), axis=0)
    return {"workload": c["desc"] + f" [strong scaling: 512 loudspeakers over {world} GPU(s)]",
            "n_gpus": world, "p50_us": pct(dev, 50), "p99_us": pct(dev, 99),
            "e2e_p99_us": pct(host, 99), "budget_us": 1e6 * c["N"] / c["fs"],
            "realtime": bool(pct(dev, 99) < 1e6 * c["N"] / c["fs"]),
            "channels": [list(p["channels"]) for p in parts],
            "k_back_bytes_per_gpu": max(p["bytes"] for p in parts),
            "definition": "max over ranks per block; device = all of a block's work, inputs in "
                          "HBM; e2e = aura_b200_process() back to back with host buffers"}


def run_b200_arm(args, cfg, rank, world, local_rank):
    import paper_2509_04390_b200 as A
    device = local_rank
    if world > 1:
        return run_sharded(args, cfg, rank, world, local_rank)
    synth, fc, mic = make_workload(cfg)
    t0 = time.perf_counter()
    eng = make_engine(A, cfg, synth, fc, device)
    t_setup = time.perf_counter() - t0
    N, Q, L = cfg["N"], cfg["Q"], cfg["L"]
    K, W = args.steps, args.warmup

    # warm-up, then device-resident timed region (value)
    eng.time_device_blocks(max(3, W), mic)
    with ClockSampler(device) as clk:
        lat_us, dev_us = eng.time_device_blocks(K, mic)
        host_us = eng.time_host_blocks(mic, K)
    clocks = clk.summary()
    phases = eng.profile_phases(min(K, 200))
    trace = eng.trace_blocks(32)
    timeline = {k: {"start_us": float(np.median(v[:, 0])), "end_us": float(np.median(v[:, 1]))}
                for k, v in trace.items()}
    peak, peak_kind = load_peaks()
    mac_name = "k_back" if phases["k_back"][1] > 0 else "k_front"
    mac_bytes = phases[mac_name][1]
    mac_us = eng.time_phase(mac_name, 20)
    achieved = mac_bytes / (mac_us * 1e-6) / 1e9
    n_launch = eng.launches_per_block()
    traffic, traffic_src = load_traffic(args.config if not args.block else None, mac_name)

    paced = None
    if not args.no_paced:
        eng.reset()  # the engine's deadline statistics cover this run only
        paced_us = eng.time_host_blocks(mic, min(K, 2000), pace_us=1e6 * N / cfg["fs"])
        dl = eng.deadline_stats()
        paced = {"p50_us": pct(paced_us, 50), "p99_us": pct(paced_us, 99),
                 "blocks": int(paced_us.size), "deadline_misses": dl["misses"], "max_us": dl["max_us"],
                 "definition": "aura_b200_process() latency with calls on the real-time grid "
                               "(one block every N/fs), host buffers"}

    cpu = None
    if not args.no_cpu_baseline:
        ref_blocks = max(3, int(args.cpu_blocks))
        L_sub, scale = cpu_sample_channels(cfg)
        us, workers, t_ref_setup = reference_blocks(cfg, synth, fc, mic, ref_blocks, 2, L_sub=L_sub)
        us = us * scale
        sub = (f"; {L_sub} of {L} loudspeakers timed and scaled x{scale:.1f} (the MAC is linear in "
               f"channels; the full reference setup alone would take minutes)") if L_sub else ""
        cpu = {"value": pct(us, 99), "unit": "us", "cores": workers, "kind": "reference",
               "p50_us": pct(us, 50),
               "sample": f"{ref_blocks} blocks of the same workload through the unmodified "
                         f"reference (oracle/_ref, ParallelBackend, -O3 -DNDEBUG); fixed-F^ "
                         f"canceller (no NLMS in the reference); setup {t_ref_setup:.1f} s excluded"
                         + sub}
    describe = eng.describe()
    del synth, fc
    eng.close()
    maxrt = None if args.no_max_rt else max_realtime(A, cfg, device, budget_s=args.max_rt_s)
    c5 = None
    if not args.no_c5:
        c5 = c5_summary([c5_secondary(A, device, K, W)], 1)

    total_bytes = sum(b for _, b in phases.values())
    # the same kernel inside the block graph (%globaltimer: first CTA start ->
    # last CTA end), concurrent with the canceller head
    # roofline regime: the working set -- spectra, canceller
    # W, delay lines -- under L2/2 stays in L2 between blocks
    P = Q if cfg["afc"] else 0
    KF = -(-cfg.get("n_hf", 0) // N) if cfg["afc"] else 0
    Kh = -(-cfg["n_h"] // N)
    footprint = 8.0 * N * (Q * L * Kh + Q * Kh + P * L * KF + (L * (KF + 1) if cfg["afc"] else 0))
    bound = roofline_regime(footprint)
    if bound == "l2":
        l2_peak, l2_kind = l2_read_peak(footprint)
        if l2_peak:
            peak, peak_kind = l2_peak, l2_kind
        else:
            bound = "hbm"
    ig = timeline.get(mac_name)
    in_graph = None
    if ig and ig["end_us"] > ig["start_us"]:
        d_us = ig["end_us"] - ig["start_us"]
        in_graph = {"us": d_us, "GBps": mac_bytes / (d_us * 1e-6) / 1e9,
                    "frac": mac_bytes / (d_us * 1e-6) / 1e9 / peak}
    line = {
        "metric": METRIC, "value": pct(dev_us, 99), "unit": "us", "n_gpus": 1,
        "steps": K, "warmup": W, "ms_per_step": float(np.mean(dev_us)) / 1000.0,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic: decaying-noise IRs (T60 = IR length, sum h^2 = 1), "
                                "AFC paths T60 0.3 s x 0.1, N(0,1) mic blocks",
        "config": {"workload": cfg["desc"], "block": N, "inputs": Q, "loudspeakers": L,
                   "taps": cfg["n_h"], "fc_taps": cfg.get("n_hf", 0),
                   "nlms_mu": cfg.get("mu", 0.0) if cfg["afc"] else None,
                   "l2": f"inputs larger than L2: {total_bytes / 1e6:.0f} MB streamed per block "
                         f"vs 126 MB L2" if total_bytes > 126e6 else
                         "working set fits L2 (real-time steady state; no flush)",
                   "parallelism": "1 GPU", "engine": describe},
        "p50_us": pct(dev_us, 50), "p99_us": pct(dev_us, 99), "max_us": float(np.max(dev_us)),
        "budget_us": 1e6 * N / cfg["fs"],
        "value_definition": "p99 device time of ALL of a block's work (its whole block graph), "
                            "back to back, inputs in HBM: CUDA events recorded by an event node "
                            "after each block graph's last kernel (end of block b-1 -> end of b)",
        "latency_to_output_us": {"p50": pct(lat_us, 50), "p99": pct(lat_us, 99),
                                 "definition": "CUDA events: graph launch -> end of k_front (which "
                                               "also runs the canceller head after publishing the "
                                               "output); the rest of the block's work follows",
                                 "published_device_us": (float(np.median(trace["output"][:, 0]))
                                                         if "output" in trace else None),
                                 "published_definition": "%globaltimer: k_front's first CTA start -> "
                                                         "the output-ready word published (median)"},
        "e2e": {"value": pct(host_us, 99), "unit": "us", "p50_us": pct(host_us, 50),
                "h2d_bytes_per_step": 4 * Q * N, "d2h_bytes_per_step": 4 * L * N,
                "path": "aura_b200_process() C-ABI, pinned mapped host I/O, back-to-back "
                        "(each call also waits for the previous block's background work)"},
        "paced_e2e": paced,
        "roofline": {"bound": bound, "kernel": mac_name, "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "footprint_bytes": footprint,
                     "peak_kind": peak_kind, "traffic": traffic, "traffic_source": traffic_src,
                     "frac_of_read_probe": achieved / READ_PROBE_GBS,
                     "bytes_per_launch": mac_bytes, "avg_launch_us": mac_us,
                     "timing": "CUDA events around 20 single launches of the kernel, back to back",
                     "in_graph": in_graph,
                     # algorithmic bytes include the canceller's W read/write and
                     # delay line, mostly L2 hits in the steady state: what HBM
                     # actually moved, from the (warm) ncu capture
                     "dram": ({"GBps": traffic / (mac_us * 1e-6) / 1e9,
                               "frac": traffic / (mac_us * 1e-6) / 1e9 / peak,
                               "frac_of_read_probe": traffic / (mac_us * 1e-6) / 1e9 / READ_PROBE_GBS}
                              if traffic and mac_us else None)},
        "phases_us_serial": {k: v[0] for k, v in phases.items()},
        "timeline_us": timeline,
        "phase_bytes": {k: v[1] for k, v in phases.items()},
        "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": int(K * n_launch),
        "max_realtime": maxrt, "c5": c5, "setup_s": t_setup,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def sharded_cfg(cfg, world, scaling):
    """Weak scaling (default): every GPU keeps the config's L loudspeakers,
    so the job has L x world; strong: the config's L is split."""
    if scaling == "weak" and world > 1:
        c = dict(cfg, L=cfg["L"] * world)
        tag = f" [weak scaling: {cfg['L']} loudspeakers per GPU x {world} GPUs]"
        c["desc"] = cfg["desc"] + tag
        if "ref_desc" in cfg:
            c["ref_desc"] = cfg["ref_desc"] + tag
        return c
    return cfg


def run_sharded(args, cfg, rank, world, local_rank):
    """N > 1: loudspeaker channels split over the ranks, one
    process per GPU. With the canceller on, the shards exchange their f^ /
    power partials every block inside the CUDA graph (k_afc_finish, P2P over
    NVLink); the synthesis shards are independent. Weak scaling by default
    (each GPU keeps the config's loudspeaker count; filter rows are generated
    per shard); --scaling strong splits the config's L. Per-block times are
    max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_2509_04390_b200 as A
    from paper_2509_04390_b200 import shard as S
    ndev = max(1, torch.cuda.device_count())
    device = local_rank % ndev
    torch.cuda.set_device(device)
    dist.init_process_group("gloo")
    cfg = sharded_cfg(cfg, world, args.scaling)
    N, Q, L = cfg["N"], cfg["Q"], cfg["L"]
    synth = LazyRows(Q * L, cfg["n_h"], cfg["fs"], seed=1000)
    fc = LazyRows(Q * L, cfg["n_hf"], cfg["fs"], t60_s=0.3, scale=0.1, seed=2000) if cfg["afc"] else None
    mic = np.random.default_rng(7).standard_normal((64, Q, N)).astype(np.float32)
    ec = A.make_config(cfg["fs"], N, Q, L, mimo=Q > 1)
    t0 = time.perf_counter()
    if cfg["afc"]:
        eng = S.ShardedAuralizer(synth, fc, ec, device=device,
                                 afc=A.AfcParams(cfg.get("mu", 0.0), 0.9, None))
        local = eng.engine
    else:
        mode = A.ChannelMode.mimo if Q > 1 else A.ChannelMode.broadcast
        eng = S.ShardedConvolver(synth, ec, world, rank, mode, device)
        local = eng.engine
    t_setup = time.perf_counter() - t0
    del synth, fc
    K, W = args.steps, args.warmup
    local.time_device_blocks(max(3, W), mic)
    dist.barrier()
    with ClockSampler(device) as clk:
        lat_us, dev_us = local.time_device_blocks(K, mic)
        dist.barrier()
        host_us = local.time_host_blocks(mic, K)
        local.synchronize()
    dist.barrier()
    clocks = clk.summary()
    phases = local.profile_phases(min(K, 200))
    mac_name = "k_back" if phases["k_back"][1] > 0 else "k_front"
    dist.barrier()
    mac_us = local.time_phase(mac_name, 20)
    mac_bytes = phases[mac_name][1]
    peak, peak_kind = load_peaks()
    n_launch = local.launches_per_block()
    dist.barrier()
    local.close()
    dist.barrier()
    # exchange ablation: the same sharded canceller with the
    # partials all-reduced by NCCL (graph-captured) instead of our P2P kernel
    nccl = None
    if cfg["afc"] and not args.no_nccl:
        # one small (P*N + 2N floats) all-reduce per block --
        # latency-bound; a pinned algorithm / protocol fixes the reduction
        # order run to run (unless the caller chose otherwise)
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "LL")
        try:
            ne = S.ShardedAuralizer(LazyRows(Q * L, cfg["n_h"], cfg["fs"], seed=1000),
                                    LazyRows(Q * L, cfg["n_hf"], cfg["fs"], t60_s=0.3, scale=0.1, seed=2000),
                                    ec, device=device, afc=A.AfcParams(cfg.get("mu", 0.0), 0.9, None),
                                    transport="nccl")
            ne.engine.time_device_blocks(max(3, W), mic)
            dist.barrier()
            _, nd = ne.engine.time_device_blocks(K, mic)
            dist.barrier()
            ne.close()
            nccl = {"dev": nd}
        except A.Error as err:
            nccl = {"error": str(err)}
        dist.barrier()
    # BASELINE configs[4]: 512 loudspeakers split over the GPUs (strong)
    c5 = None if args.no_c5 else c5_secondary(A, device, K, W, world, rank)
    dist.barrier()
    # max real time per GPU (c3 shape, each GPU on its own: needs a device
    # per rank), summed over the GPUs
    maxrt = None
    if not args.no_max_rt and ndev >= world:
        maxrt = max_realtime(A, dict(CONFIGS[args.config]), device, budget_s=args.max_rt_s)
    dist.barrier()
    mine = {"lat": lat_us, "dev": dev_us, "host": host_us, "mac_us": mac_us, "nccl": nccl,
            "mac_bytes": mac_bytes, "launches": n_launch, "c5": c5, "maxrt": maxrt,
            "clocks": clocks, "channels": (eng.l0, eng.l1), "setup": t_setup}
    allr = [None] * world
    dist.all_gather_object(allr, mine)
    if rank == 0:
        dev = np.max(np.stack([r["dev"] for r in allr]), axis=0)
        lat = np.max(np.stack([r["lat"] for r in allr]), axis=0)
        host = np.max(np.stack([r["host"] for r in allr]), axis=0)
        slowest = max(allr, key=lambda r: r["mac_us"])
        achieved = slowest["mac_bytes"] / (slowest["mac_us"] * 1e-6) / 1e9
        line = {
            "metric": METRIC, "value": pct(dev, 99), "unit": "us", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": float(np.mean(dev)) / 1000.0,
            "higher_is_better": False, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic: decaying-noise IRs, N(0,1) mic blocks",
            "config": {"workload": cfg["desc"], "block": N, "inputs": Q, "loudspeakers": L,
                       "taps": cfg["n_h"], "fc_taps": cfg.get("n_hf", 0),
                       "parallelism": f"{world} GPUs, loudspeaker channels sharded "
                                      f"{[r['channels'] for r in allr]}",
                       "exchange": "P2P NVLink stores + system-scope flags in k_afc_finish "
                                   "(P*N + 2N floats per block)" if cfg["afc"] else "none",
                       "devices_visible": ndev},
            "p50_us": pct(dev, 50), "p99_us": pct(dev, 99), "budget_us": 1e6 * N / cfg["fs"],
            "value_definition": "p99 over blocks of the max over ranks of the device time of "
                                "all of a block's work",
            "latency_to_output_us": {"p50": pct(lat, 50), "p99": pct(lat, 99)},
            "e2e": {"value": pct(host, 99), "unit": "us", "p50_us": pct(host, 50),
                    "h2d_bytes_per_step": 4 * Q * N * world,
                    "d2h_bytes_per_step": 4 * L * N},
            "roofline": {"bound": "hbm", "kernel": mac_name, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "peak_kind": peak_kind,
                         "traffic": None, "bytes_per_launch": slowest["mac_bytes"],
                         "avg_launch_us": slowest["mac_us"], "per": "slowest rank"},
            "cpu_baseline": None, "clocks": allr[0]["clocks"],
            "gpu_launches": int(K * sum(r["launches"] for r in allr)),
            "setup_s": max(r["setup"] for r in allr),
            "c5": c5_summary([r["c5"] for r in allr], world) if allr[0]["c5"] else None,
            "exchange_ablation": _exchange_ablation(dev, allr),
            "max_realtime": ({"channels": sum(r["maxrt"]["channels"] for r in allr),
                              "taps": cfg["n_h"],
                              "channels_x_taps": sum(r["maxrt"]["channels"] for r in allr) * cfg["n_h"],
                              "per_gpu_channels": [r["maxrt"]["channels"] for r in allr],
                              "criteria": "per GPU: device block p99 AND paced process() e2e p99 "
                                          "< N/f_s (c3 shape on each GPU; the cross-GPU canceller "
                                          "exchange is timed in value)"}
                             if all(r["maxrt"] for r in allr) else None),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def _exchange_ablation(dev_p2p, allr):
    """Block p50/p99 (max over ranks) with the P2P exchange kernel (value)
    and with the NCCL all-reduce, or why NCCL did not run."""
    if not allr[0]["nccl"]:
        return None
    errs = [r["nccl"]["error"] for r in allr if "error" in r["nccl"]]
    out = {"p2p": {"p50_us": pct(dev_p2p, 50), "p99_us": pct(dev_p2p, 99)},
           "nccl_env": {k: os.environ.get(k) for k in ("NCCL_ALGO", "NCCL_PROTO")}}
    if errs:
        out["nccl"] = {"error": errs[0]}
    else:
        nd = np.max(np.stack([r["nccl"]["dev"] for r in allr]), axis=0)
        out["nccl"] = {"p50_us": pct(nd, 50), "p99_us": pct(nd, 99)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--block", type=int, default=None, help="override block size (c4 sweep)")
    ap.add_argument("--cpu-blocks", type=int, default=60)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-max-rt", action="store_true", help="skip the max real-time search")
    ap.add_argument("--max-rt-s", type=float, default=110.0, help="time box of the max-RT search")
    ap.add_argument("--no-c5", action="store_true", help="skip the configs[4] (c5) line")
    ap.add_argument("--no-nccl", action="store_true", help="N > 1: skip the NCCL exchange ablation")
    ap.add_argument("--no-paced", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak keeps the config's loudspeakers per GPU, strong splits them")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.block:
        cfg["N"] = args.block
        cfg["desc"] += f" [block {args.block}]"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, cfg, rank)
    return run_b200_arm(args, cfg, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
