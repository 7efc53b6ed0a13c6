"""Small workload for compute-sanitizer (tests/test_gpu_sanitizer.py): every
kernel of the product on smoke-sized engines -- a broadcast convolver, an
elementwise convolver, an NLMS auralizer (fused head and the separate
k_back_head), a MIMO auralizer, virtual shards (k_afc_finish), the stream
launch mode and the measurement relaunches. Exits non-zero on a parity miss."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
import paper_2509_04390_b200 as A  # noqa: E402
from paper_2509_04390_b200 import shard as S  # noqa: E402
from conftest import decaying_filters, rel_err  # noqa: E402


def check(y, ref, what):
    err = rel_err(y, ref)
    if not err <= 1e-5:
        print(f"PARITY {what}: {err:.3e}")
        sys.exit(3)


def main():
    print("library:", A.lib()._name, flush=True)
    rng = np.random.default_rng(1)
    N = 64
    # broadcast convolver, then the stream launch mode
    f = decaying_filters(rng, 8, 20 * N)
    c = A.Convolver(list(f), A.make_config(48000, N, 1, 8))
    o = O.OracleConvolver(f, N, 1, 8, O.BROADCAST)
    for b in range(12):
        if b == 6:
            c.set_launch_mode(1)
        x = rng.standard_normal((1, N)).astype(np.float32)
        check(c.process(x), o.process(x), "broadcast")
    c.time_phase("k_back", 2)
    c.close()
    # elementwise
    fe = decaying_filters(rng, 4, 7 * 32)
    ce = A.Convolver(list(fe), A.make_config(48000, 32, 4, 4), A.ChannelMode.elementwise)
    oe = O.OracleConvolver(fe, 32, 4, 4, O.ELEMENTWISE)
    for _ in range(10):
        x = rng.standard_normal((4, 32)).astype(np.float32)
        check(ce.process(x), oe.process(x), "elementwise")
    ce.close()
    # NLMS auralizer (fused head), MIMO, k_back_head (env knob), and the
    # constrained update (k_afc_constrain)
    for Q, L, fused, cons in ((1, 8, True, False), (2, 6, True, False), (1, 8, False, False),
                              (1, 8, True, True), (2, 6, False, True)):
        os.environ["AURA_B200_FRONT_HEAD"] = "1" if fused else "0"
        s = decaying_filters(rng, Q * L, 9 * N, scale=0.5)
        fc = decaying_filters(rng, Q * L, 3 * N, scale=0.1)
        kw = dict(gain=0.9, mu=0.02, lam=0.9, delta=1e-2)
        g = A.Auralizer(list(s), list(fc), A.make_config(48000, N, Q, L, mimo=Q > 1), input_gain=0.9,
                        afc=A.AfcParams(0.02, 0.9, 1e-2, cons))
        oa = O.OracleAuralizer(s, fc, N, Q, L, constrained=cons, **kw)
        for _ in range(10):
            m = rng.standard_normal((Q, N)).astype(np.float32)
            check(g.process(m), oa.process(m), f"auralizer Q={Q} fused={fused} constrained={cons}")
        check(g.coeffs(), oa.coeffs(), "W")
        g.time_device_blocks(3)
        g.time_phase("k_front", 2)
        g.trace_blocks(2)
        g.close()
    os.environ.pop("AURA_B200_FRONT_HEAD", None)
    # virtual shards: the canceller exchange (k_afc_finish)
    s = decaying_filters(rng, 8, 9 * N, scale=0.5)
    fc = decaying_filters(rng, 8, 3 * N, scale=0.1)
    v = S.VirtualShards(list(s), list(fc), A.make_config(48000, N, 1, 8), 2,
                        afc=A.AfcParams(0.02, 0.9, 1e-2))
    ov = O.OracleAuralizer(s, fc, N, 1, 8, mu=0.02, lam=0.9, delta=1e-2)
    for _ in range(8):
        m = rng.standard_normal((1, N)).astype(np.float32)
        check(v.process(m), ov.process(m), "virtual shards")
    v.close()
    print("sanitize workload: ok")


if __name__ == "__main__":
    main()
