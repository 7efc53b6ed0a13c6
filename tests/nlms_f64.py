"""Independent float64 restatement of SURVEY.md Appendix A (PBFDAF/NLMS
canceller) + Appendix B (MIMO) with numpy FFTs. Used only to validate the C
oracle's adaptation path, which has no reference implementation."""
import numpy as np


class NlmsF64:
    def __init__(self, synth, fc, N, Q, L, gain=1.0, mu=0.0, lam=0.9, delta=None, constrained=False):
        self.N, self.Q, self.L = N, Q, L
        self.constrained = constrained
        self.gain, self.mu, self.lam = gain, mu, lam
        self.delta = 1e-6 * N if delta is None else delta
        synth = np.asarray(synth, np.float64).reshape(Q, L, -1)
        fc = np.asarray(fc, np.float64).reshape(Q, L, -1)
        self.K = -(-synth.shape[2] // N)
        self.KF = -(-fc.shape[2] // N)
        self.H = self._part(synth, self.K)      # Q,L,K,bins
        self.W = self._part(fc, self.KF)        # P,L,KF,bins
        self.Xin = np.zeros((Q, self.K, N + 1), complex)   # age-ordered
        self.Xa = np.zeros((L, self.KF, N + 1), complex)
        self.win = np.zeros((Q, 2 * N))
        self.swin = np.zeros((L, 2 * N))
        self.fhat = np.zeros((Q, N))
        self.power = np.zeros(N + 1)

    def _part(self, taps, K):
        N = self.N
        pad = np.zeros(taps.shape[:-1] + (K * N,))
        pad[..., :taps.shape[-1]] = taps
        blocks = pad.reshape(taps.shape[:-1] + (K, N))
        z = np.concatenate([blocks, np.zeros_like(blocks)], axis=-1)
        return np.fft.rfft(z, axis=-1)

    def process(self, mic):
        N = self.N
        mt = self.gain * np.asarray(mic, np.float64).reshape(self.Q, N) - self.fhat
        if self.mu != 0.0:
            E = np.fft.rfft(np.concatenate([np.zeros((self.Q, N)), mt], axis=1), axis=1)
            scale = self.mu / (self.power + self.delta)
            G = scale * np.conj(self.Xa)[None] * E[:, None, None, :]
            if self.constrained:  # App. A step 2: keep the first N taps of the gradient
                g = np.fft.irfft(G, n=2 * N, axis=-1)
                g[..., N:] = 0.0
                G = np.fft.rfft(g, axis=-1)
            self.W += G
        self.win = np.concatenate([self.win[:, N:], mt], axis=1)
        self.Xin = np.concatenate([np.fft.rfft(self.win, axis=1)[:, None], self.Xin[:, :-1]], axis=1)
        Y = np.einsum("qkj,qlkj->lj", self.Xin, self.H)
        spk = np.fft.irfft(Y, n=2 * N, axis=1)[:, N:]
        self.swin = np.concatenate([self.swin[:, N:], spk], axis=1)
        self.Xa = np.concatenate([np.fft.rfft(self.swin, axis=1)[:, None], self.Xa[:, :-1]], axis=1)
        Yf = np.einsum("lkj,plkj->pj", self.Xa, self.W)
        self.fhat = np.fft.irfft(Yf, n=2 * N, axis=1)[:, N:]
        if self.mu != 0.0:
            s = np.sum(np.abs(self.Xa[:, 0]) ** 2, axis=0)
            self.power = self.lam * self.power + (1 - self.lam) * s
        return spk

    def feedback_estimate(self):
        return self.fhat
