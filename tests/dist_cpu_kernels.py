"""Numpy shard kernels for the CPU/gloo tests of paper_2003_07020_b200.distributed (TEST ONLY).

They restate the per-rank math of the reference (all_at_once.hpp:33-55 with a dense Jacobian,
alpha_circulant.hpp:146-198 time FFTs on a column shard, tau.hpp:98-119 on a frequency-row shard)
so the sharding/communication logic of ShardedSolver can be checked against the single-process
oracle without a GPU.  Never used on the product path.
"""
import numpy as np
import torch


def dst_matrix(n):
    i = np.arange(1, n + 1)
    return np.sqrt(2.0 / (n + 1)) * np.sin(np.pi * np.outer(i, i) / (n + 1))


def toeplitz(col):
    n = len(col)
    idx = np.abs(np.arange(n)[:, None] - np.arange(n)[None, :])
    return np.asarray(col)[idx]


class NumpyShardKernels:
    device = torch.device("cpu")

    def __init__(self, po, nt, dt, two_dim, n):
        self.nt, self.dt, self.H = nt, dt, nt // 2 + 1
        lam = po.lam()
        self.lam = lam
        self.sigma = po.sigma()
        a = po.alpha
        k = np.arange(nt) / nt
        self.sf, self.sb = a ** k, a ** (-k)
        if two_dim:
            wx, wy = po.column(0), po.column(1)
            sx, sy = po.scales
            self.A = -sx * np.kron(toeplitz(wx), np.eye(n)) - sy * np.kron(np.eye(n), toeplitz(wy))
            Q = dst_matrix(n)
            self.Q = np.kron(Q, Q)
        else:
            self.A = toeplitz(po.column(0))
            self.Q = dst_matrix(n)
        self.ns = self.A.shape[0]

    def empty(self, n, complex_=False):
        return torch.empty(n, dtype=torch.complex128 if complex_ else torch.float64)

    def matvec(self, buf, nt_local, koff, halo):
        ns, arr = self.ns, buf.numpy()
        base = 2 * ns if halo else 0
        y = np.empty(nt_local * ns)
        for k in range(nt_local):
            kg = koff + k
            vk = arr[base + k * ns: base + (k + 1) * ns]
            c = vk.copy()
            if kg >= 1:
                c = 1.5 * vk + -2.0 * arr[base + (k - 1) * ns: base + k * ns]
            if kg >= 2:
                c = c + 0.5 * arr[base + (k - 2) * ns: base + (k - 1) * ns]
            y[k * ns:(k + 1) * ns] = c - self.dt * (self.A @ vk)
        return torch.from_numpy(y)

    def time_fwd(self, cols, ns_local, s_in):
        X = cols.numpy().reshape(self.nt, ns_local) * (self.sf[:, None] * s_in)
        R = np.fft.ifft(X, axis=0) * self.nt  # e^{+2 pi i kn/Nt} (alpha_circulant.hpp:150)
        return torch.from_numpy(np.ascontiguousarray(R[:self.H]).ravel())

    def tau(self, Zrows, row0, nrows, forward=False):
        Z = Zrows.numpy().reshape(nrows, self.ns)  # shares memory with the tensor
        for r in range(nrows):
            d = self.lam[row0 + r] - self.dt * self.sigma
            t = self.Q @ Z[r]
            Z[r] = self.Q @ (t * d if forward else t / d)

    def time_inv(self, Z, ns_local):
        Zh = Z.numpy().reshape(self.H, ns_local)
        F = np.empty((self.nt, ns_local), complex)
        F[:self.H] = Zh
        for n in range(self.H, self.nt):
            F[n] = np.conj(Zh[self.nt - n])
        z = np.fft.fft(F, axis=0).real * (self.sb / self.nt)[:, None]
        return torch.from_numpy(np.ascontiguousarray(z).ravel())

    # commuted ordering (1D): S per time level; per-column time solve over all Nt frequencies
    def dst_levels(self, v, nt_local, s_in):
        X = v.numpy().reshape(nt_local, self.ns)
        return torch.from_numpy(np.ascontiguousarray((X @ self.Q.T) * s_in).ravel())

    def time_solve(self, cols, col0, ns_local, forward=False):
        X = cols.numpy().reshape(self.nt, ns_local) * self.sf[:, None]
        F = np.fft.ifft(X, axis=0) * self.nt  # e^{+2 pi i kn/Nt}
        lam = np.empty(self.nt, complex)
        lam[:self.H] = self.lam[:self.H]
        for n in range(self.H, self.nt):
            lam[n] = np.conj(self.lam[self.nt - n])
        d = lam[:, None] - self.dt * self.sigma[None, col0:col0 + ns_local]
        Y = F * d if forward else F / d
        z = np.fft.fft(Y, axis=0).real * (self.sb / self.nt)[:, None]
        return torch.from_numpy(np.ascontiguousarray(z).ravel())

    def dots(self, V, scales, w, with_norm):
        wn = w.numpy()
        out = [s * float(v.numpy() @ wn) for v, s in zip(V, scales)]
        if with_norm or not V:
            out.append(float(wn @ wn))
        return np.array(out)

    def update(self, V, coef, w):
        wn = w.numpy()
        for v, c in zip(V, coef):
            wn -= c * v.numpy()
        return float(wn @ wn)

    def lincomb(self, V, coef):
        u = np.zeros(V[0].numel())
        for v, c in zip(V, coef):
            u += c * v.numpy()
        return torch.from_numpy(u)
