"""Host FP64 restatement of the distributed engine's per-rank block steps -- TEST
INFRASTRUCTURE (built on the oracle; never imported by the package).  It mirrors the C-ABI
``mle_dctx_*`` semantics (paper_2601_11437_b200/distributed.py) with FP64 numpy panels so that
the driver, its ownership rules and its collectives are tested with gloo on CPU."""

import math

import numpy as np

BLOCK = 512


class HostPanels:
    """The same block algorithm in FP64 numpy (host), for testing the driver on CPU."""

    def __init__(self, locations, values, rank, world, nugget=0.0):
        self.loc = np.asarray(locations, float)
        self.z = np.asarray(values, float)
        self.n = self.loc.shape[0]
        self.rank, self.world = rank, world
        self.nugget = float(nugget)
        self.N = -(-(self.n + 1) // BLOCK) * BLOCK
        self.nb = self.N // BLOCK
        self.nmat = 3 if self.nugget > 0.0 else 2
        self.owned = list(range(rank, self.nb, world))
        self.W = {}

    def close(self):
        pass

    def exchange(self, kind):
        import torch

        N = self.N
        size = {"P": (N - BLOCK) * BLOCK, "W": N * BLOCK, "X": self.nmat * N * BLOCK}[kind]
        return torch.zeros(size, dtype=torch.float64)

    def _full(self, theta, kind):
        from oracle import maternmle_cpu as O  # host test backend only (tests/, CPU)

        n, N = self.n, self.N
        out = np.zeros((N, N))
        if kind == "sigma":
            out[:n, :n] = O.matrix(self.loc, theta, "sigma", self.nugget)
            out[n, :n] = self.z
            out[:n, n] = self.z
            idx = np.arange(n + 1, N)
            out[idx, idx] = 1.0
        elif kind == "ident":
            out[np.arange(n), np.arange(n)] = 1.0
        else:
            out[:n, :n] = O.matrix(self.loc, theta, kind)
        return out

    def begin(self, theta, derivs):
        self.derivs = bool(derivs)
        self.fail, self.pivot = 0, 0
        cols = lambda m: {b: m[:, b * BLOCK:(b + 1) * BLOCK].copy() for b in self.owned}
        self.sig = cols(self._full(theta, "sigma"))
        if self.derivs:
            kinds = ["alpha", "nu"] + (["ident"] if self.nmat == 3 else [])
            self.mat = [cols(self._full(theta, k)) for k in kinds]

    def factor(self, b, exch):
        c0, c1, N, n = b * BLOCK, (b + 1) * BLOCK, self.N, self.n
        p = self.sig[b]
        for j in range(BLOCK):  # column-by-column Cholesky of the block (all rows)
            g = c0 + j
            col = p[g:, j] - p[g:, :j] @ p[g, :j]
            if g == n:
                piv = 1.0  # augmented index: row n carries y = L^-1 z, no pivot check
            elif not (col[0] > 0.0) and not self.fail:
                self.fail, self.pivot = 1, g
                piv = 1.0
            else:
                piv = math.sqrt(col[0]) if col[0] > 0.0 else 1.0
            p[g, j] = piv
            p[g + 1:, j] = col[1:] / piv
            p[c0:g, j] = 0.0
        if c1 < N:
            exch.view(-1)[: (N - c1) * BLOCK] = \
                __import__("torch").from_numpy(np.ascontiguousarray(p[c1:, :]).ravel())

    def update(self, b, exch, lo=0, hi=None):
        hi = self.nb if hi is None else hi
        c1, N = (b + 1) * BLOCK, self.N
        P = exch.numpy()[: (N - c1) * BLOCK].reshape(N - c1, BLOCK)
        for j in self.owned:
            if j <= b or not lo <= j < hi:
                continue
            cj = j * BLOCK
            Pj = P[cj - c1:, :]
            self.sig[j][cj:, :] -= Pj @ P[cj - c1:cj - c1 + BLOCK, :].T

    def wcache(self, on=True):
        self.cache_w = bool(on)
        self.wc = {}
        return self.cache_w

    def wblock(self, b, exch):
        import scipy.linalg as sla

        c0, c1, N = b * BLOCK, (b + 1) * BLOCK, self.N
        p = self.sig[b]
        dinv = sla.solve_triangular(p[c0:c1, :], np.eye(BLOCK), lower=True)
        w = np.vstack([dinv, -p[c1:, :] @ dinv])
        self.W[b] = w
        self.Dinv = getattr(self, "Dinv", {})
        self.Dinv[b] = dinv
        if exch is not None:
            exch.view(-1)[: (N - c0) * BLOCK] = __import__("torch").from_numpy(w.ravel())

    # two-sided reduction (the sygst recurrence) on the panels, FP64
    def ts_owner(self, b, exch_x):
        c0, c1, N = b * BLOCK, (b + 1) * BLOCK, self.N
        dinv, L21 = self.Dinv[b], self.sig[b][c1:, :]
        self.S11 = getattr(self, "S11", {})
        buf = exch_x.numpy().reshape(self.nmat, N * BLOCK)
        for m, mats in enumerate(self.mat):
            s11 = dinv @ mats[b][c0:c1, :] @ dinv.T
            mats[b][c0:c1, :] = s11
            self.S11[(b, m)] = s11
            if c1 < N:
                s21 = mats[b][c1:, :] @ dinv.T - 0.5 * L21 @ s11
                mats[b][c1:, :] = s21
                buf[m, : (N - c1) * BLOCK] = s21.ravel()

    def ts_finish(self, b):
        c1 = (b + 1) * BLOCK
        for m, mats in enumerate(self.mat):
            if c1 < self.N:
                mats[b][c1:, :] -= 0.5 * self.sig[b][c1:, :] @ self.S11[(b, m)]

    def ts_update(self, b, exch_x, exch_p, lo=0, hi=None):
        hi = self.nb if hi is None else hi
        c1, N = (b + 1) * BLOCK, self.N
        L = exch_p.numpy()[: (N - c1) * BLOCK].reshape(N - c1, BLOCK)
        xs = exch_x.numpy().reshape(self.nmat, N * BLOCK)
        for m, mats in enumerate(self.mat):
            S = xs[m, : (N - c1) * BLOCK].reshape(N - c1, BLOCK)
            for j in self.owned:
                if j <= b or not lo <= j < hi:
                    continue
                r = j * BLOCK - c1
                mats[j][j * BLOCK:, :] -= S[r:] @ L[r:r + BLOCK].T + L[r:] @ S[r:r + BLOCK].T

    def panel_slices(self, b, exch_p):
        c1, N = (b + 1) * BLOCK, self.N
        if c1 < N:
            exch_p.view(-1)[: (N - c1) * BLOCK] = \
                __import__("torch").from_numpy(np.ascontiguousarray(self.sig[b][c1:, :]).ravel())

    def forward(self, b, exch, lo=0, hi=None):
        hi = self.nb if hi is None else hi
        c0, c1, N = b * BLOCK, (b + 1) * BLOCK, self.N
        w = exch.numpy()[: (N - c0) * BLOCK].reshape(N - c0, BLOCK)
        if getattr(self, "cache_w", False):
            self.wc[b] = w.copy()
        for mats in self.mat:
            for j in self.owned:
                if not lo <= j < hi:
                    continue
                x = mats[j][c0:c1, :].copy()
                mats[j][c0:c1, :] = w[:BLOCK] @ x
                mats[j][c1:, :] += w[BLOCK:] @ x

    def right_operand(self, b, exch):
        c0, N = b * BLOCK, self.N
        buf = exch.numpy().reshape(self.nmat, N * BLOCK)
        for m, mats in enumerate(self.mat):
            a = mats[b][c0:, :].copy()
            a[np.triu_indices(BLOCK, 1)] = 0.0  # only k <= r (rows and columns from c0)
            buf[m, : (N - c0) * BLOCK] = a.ravel()

    def right(self, b, exch_w, exch_x, lo=0, hi=None):
        hi = self.nb if hi is None else hi
        c0, N = b * BLOCK, self.N
        if exch_w is None:
            w = self.wc[b]
        else:
            w = exch_w.numpy()[: (N - c0) * BLOCK].reshape(N - c0, BLOCK)
        xs = exch_x.numpy().reshape(self.nmat, N * BLOCK)
        for m, mats in enumerate(self.mat):
            x = xs[m, : (N - c0) * BLOCK].reshape(N - c0, BLOCK)
            for j in self.owned:
                if j < b or not lo <= j < hi:
                    continue
                cj = j * BLOCK
                upd = x[cj - c0:, :] @ w[cj - c0:cj - c0 + BLOCK, :].T
                if j == b:
                    mats[j][cj:, :] = upd
                else:
                    mats[j][cj:, :] += upd

    def partials(self):
        n = self.n
        s = np.zeros(16)
        for b in self.owned:
            c0 = b * BLOCK
            L = self.sig[b]
            for jl in range(BLOCK):
                j = c0 + jl
                if j < n:
                    s[0] += math.log(L[j, jl])
                    s[1] += L[n, jl] ** 2
                    if self.derivs:
                        a, c = self.mat[0][b][j:n, jl], self.mat[1][b][j:n, jl]
                        wgt = np.full(a.shape, 2.0)
                        wgt[0] = 1.0
                        s[2] += a[0]
                        s[3] += c[0]
                        s[4] += np.sum(wgt * a * a)
                        s[5] += np.sum(wgt * a * c)
                        s[6] += np.sum(wgt * c * c)
                        if self.nmat == 3:
                            mm = self.mat[2][b][j:n, jl]
                            s[7] += mm[0]
                            s[8] += np.sum(wgt * a * mm)
                            s[9] += np.sum(wgt * c * mm)
                            s[10] += np.sum(wgt * mm * mm)
                if j == n and self.derivs:
                    s[11] = self.mat[0][b][n, jl]
                    s[12] = self.mat[1][b][n, jl]
                    if self.nmat == 3:
                        s[13] = self.mat[2][b][n, jl]
        s[14], s[15] = float(self.fail), float(self.pivot)
        return s
