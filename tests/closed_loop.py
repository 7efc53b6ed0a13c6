"""Closed-loop acoustic feedback simulator -- restates the reference's
oracle::simulate_closed_loop (oracle.hpp:58-122) for any auralizer object
with process(mic (Q,N)) -> (L,N) and feedback_estimate() -> (Q,N).

The physical feedback is computed in float64 with direct convolution on the
loudspeaker history (never with the engine under test); the response of
l_n starts at timeline index (n+1)*N, the estimate alignment the reference
uses (auralizer.hpp:21-23), so F^ = F cancels exactly."""
import numpy as np


def simulate(aur, source, true_paths, N, blocks, gain=1.0):
    """source: (Q, >= blocks*N) float64; true_paths: (P=Q, L, n_f) float64.
    Returns dict(mic, speakers, residual) lists per block."""
    Q = source.shape[0]
    L = true_paths.shape[1]
    max_path = true_paths.shape[2]
    timeline = np.zeros((Q, (blocks + 1) * N + max_path))
    mic_blocks, spk_blocks, res_blocks = [], [], []
    for n in range(blocks):
        mic = (source[:, n * N:(n + 1) * N] + timeline[:, n * N:(n + 1) * N]).astype(np.float32)
        mic_blocks.append(mic)
        est = np.asarray(aur.feedback_estimate(), np.float32).reshape(Q, N)
        res = gain * mic - est - source[:, n * N:(n + 1) * N].astype(np.float32)
        res_blocks.append(res)
        spk = np.asarray(aur.process(mic), np.float32)
        spk_blocks.append(spk)
        off = (n + 1) * N
        for p in range(Q):
            for l in range(L):
                r = np.convolve(spk[l].astype(np.float64), true_paths[p, l])
                end = min(off + r.size, timeline.shape[1])
                timeline[p, off:end] += r[:end - off]
    return dict(mic=mic_blocks, speakers=spk_blocks, residual=res_blocks)
