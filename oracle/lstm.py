"""ORACLE / TEST INFRASTRUCTURE ONLY — numpy restatement of the reference's
stacked-LSTM demand predictor (src/lstm.cpp, include/lorasim/lstm.hpp) and
its online wrapper's bookkeeping (src/predictor.cpp).

The reference's lstm.cpp needs Eigen3 (absent here), so it cannot be
compiled; this port follows its batched matrix formulation line by line and
is itself pinned against the reference's Eigen-free scalar test oracle
(tests/support/lstm_reference.hpp via oracle/_ref/libref.so) and central
finite differences, exactly as tests/test_predictor.cpp:72-110 does.
"""
from __future__ import annotations

import numpy as np

CLAMP = 1e-7  # lstm.cpp:12


def _sigmoid(x):  # lstm.cpp:14-18 (stable form)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def clamped_ce(p, y):  # lstm.cpp:24-27
    q = np.clip(p, CLAMP, 1.0 - CLAMP)
    return -(y * np.log(q) + (1.0 - y) * np.log(1.0 - q))


class Layout:
    """Flat θ layout (lstm.cpp:59-76)."""

    def __init__(self, window, hidden, layers, embedding_dim, num_adapters):
        self.T, self.H, self.L, self.E, self.A = window, hidden, layers, embedding_dim, num_adapters
        self.in0 = 1 + embedding_dim
        off = 0
        self.w_off, self.u_off, self.b_off = [], [], []
        for l in range(layers):
            inp = self.in0 if l == 0 else hidden
            self.w_off.append(off)
            off += 4 * hidden * inp
            self.u_off.append(off)
            off += 4 * hidden * hidden
            self.b_off.append(off)
            off += 4 * hidden
        self.head_w, self.head_b = off, off + hidden
        off += hidden + 1
        self.emb = off
        off += embedding_dim * num_adapters
        self.size = off

    def mats(self, theta, l):
        H = self.H
        inp = self.in0 if l == 0 else H
        W = theta[self.w_off[l]:self.w_off[l] + 4 * H * inp].reshape(inp, 4 * H).T  # column-major
        U = theta[self.u_off[l]:self.u_off[l] + 4 * H * H].reshape(H, 4 * H).T
        b = theta[self.b_off[l]:self.b_off[l] + 4 * H]
        return W, U, b


def _logits(lay: Layout, theta, adapters, windows, cache=None):
    """lstm.cpp:87-170: H×B matrices per timestep."""
    H, T, E = lay.H, lay.T, lay.E
    B = len(adapters)
    emb = theta[lay.emb:lay.emb + E * lay.A].reshape(lay.A, E).T  # E × A
    emb_cols = emb[:, adapters]
    layer_in = []
    for t in range(T):
        x = np.empty((lay.in0, B))
        x[0] = windows[:, t]
        x[1:] = emb_cols
        layer_in.append(x)
    if cache is not None:
        cache["x0"] = [x.copy() for x in layer_in]
        for k in ("i", "f", "g", "o", "c", "tc", "h"):
            cache[k] = [[] for _ in range(lay.L)]
    for l in range(lay.L):
        W, U, b = lay.mats(theta, l)
        h = np.zeros((H, B))
        c = np.zeros((H, B))
        for t in range(T):
            z = W @ layer_in[t] + U @ h + b[:, None]
            i, f = _sigmoid(z[:H]), _sigmoid(z[H:2 * H])
            g, o = np.tanh(z[2 * H:3 * H]), _sigmoid(z[3 * H:])
            c = f * c + i * g
            tc = np.tanh(c)
            h = o * tc
            if cache is not None:
                for k, v in (("i", i), ("f", f), ("g", g), ("o", o), ("c", c), ("tc", tc), ("h", h)):
                    cache[k][l].append(v)
            layer_in[t] = h
    head_w = theta[lay.head_w:lay.head_w + H]
    return head_w @ layer_in[T - 1] + theta[lay.head_b]


def forward(lay, theta, adapters, windows):  # lstm.cpp:172-175
    return _sigmoid(_logits(lay, theta, np.asarray(adapters), np.asarray(windows, dtype=float)))


def loss_on(lay, theta, adapters, windows, labels):  # lstm.cpp:185-190
    p = forward(lay, theta, adapters, windows)
    return float(clamped_ce(p, np.asarray(labels, dtype=float)).sum() / len(adapters))


def gradient(lay, theta, adapters, windows, labels):
    """BPTT, lstm.cpp:192-281."""
    adapters = np.asarray(adapters)
    windows = np.asarray(windows, dtype=float)
    labels = np.asarray(labels, dtype=float)
    H, T, E, B = lay.H, lay.T, lay.E, len(adapters)
    cache = {}
    z = _logits(lay, theta, adapters, windows, cache)
    grad = np.zeros(lay.size)
    dlogit = (_sigmoid(z) - labels) / B
    head_w = theta[lay.head_w:lay.head_w + H]
    grad[lay.head_w:lay.head_w + H] = cache["h"][lay.L - 1][T - 1] @ dlogit
    grad[lay.head_b] = dlogit.sum()
    dh_ext = [np.zeros((H, B)) for _ in range(T)]
    dh_ext[T - 1] = np.outer(head_w, dlogit)
    for l in range(lay.L - 1, -1, -1):
        W, U, _ = lay.mats(theta, l)
        inp = W.shape[1]
        gW = np.zeros((4 * H, inp))
        gU = np.zeros((4 * H, H))
        gb = np.zeros(4 * H)
        dx_below = [None] * T
        dc_next = np.zeros((H, B))
        dh_carry = np.zeros((H, B))
        for t in range(T - 1, -1, -1):
            i, f, g, o = (cache[k][l][t] for k in ("i", "f", "g", "o"))
            tc = cache["tc"][l][t]
            dh = dh_ext[t] + dh_carry
            dO = dh * tc
            dc = dc_next + dh * o * (1.0 - tc * tc)
            di, dg = dc * g, dc * i
            c_prev = cache["c"][l][t - 1] if t > 0 else np.zeros((H, B))
            df = dc * c_prev
            dc_next = dc * f
            dz = np.concatenate([di * i * (1 - i), df * f * (1 - f), dg * (1 - g * g),
                                 dO * o * (1 - o)])
            x_t = cache["x0"][t] if l == 0 else cache["h"][l - 1][t]
            h_prev = cache["h"][l][t - 1] if t > 0 else np.zeros((H, B))
            gW += dz @ x_t.T
            gU += dz @ h_prev.T
            gb += dz.sum(axis=1)
            dh_carry = U.T @ dz
            dx_below[t] = W.T @ dz
        grad[lay.w_off[l]:lay.w_off[l] + gW.size] = gW.T.reshape(-1)
        grad[lay.u_off[l]:lay.u_off[l] + gU.size] = gU.T.reshape(-1)
        grad[lay.b_off[l]:lay.b_off[l] + 4 * H] = gb
        if l > 0:
            dh_ext = dx_below
        else:
            g_emb = grad[lay.emb:lay.emb + E * lay.A].reshape(lay.A, E)
            for t in range(T):
                for b in range(B):
                    g_emb[adapters[b]] += dx_below[t][1:, b]
    return grad


class Adam:
    """PredictorModel::train_step's Adam update (lstm.cpp:283-296)."""

    def __init__(self, n, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        self.m, self.v, self.t = np.zeros(n), np.zeros(n), 0
        self.lr, self.b1, self.b2, self.eps = lr, b1, b2, eps

    def step(self, theta, g):
        self.t += 1
        self.m = self.b1 * self.m + (1 - self.b1) * g
        self.v = self.b2 * self.v + (1 - self.b2) * g * g
        mc = 1 - self.b1 ** self.t
        vc = 1 - self.b2 ** self.t
        theta -= self.lr * (self.m / mc) / (np.sqrt(self.v / vc) + self.eps)


def init_theta(lay: Layout, seed: int) -> np.ndarray:
    """mt19937_64(seed) + uniform_real_distribution(-1/√H, 1/√H) (lstm.cpp:77-81).

    libstdc++'s uniform_real_distribution<double> draws one 64-bit word and
    maps it through generate_canonical: u = x / 2^64; value = a + (b - a)·u."""
    from .mt64 import MT19937_64
    rng = MT19937_64(seed)
    bound = 1.0 / np.sqrt(float(lay.H))
    out = np.empty(lay.size)
    for k in range(lay.size):
        u = float(rng.next()) / 18446744073709551616.0
        if u >= 1.0:
            u = np.nextafter(1.0, 0.0)
        out[k] = (bound - -bound) * u + -bound
    return out


def normalized_window(ring, run_max, window):  # predictor.cpp:52-60
    out = np.zeros(window)
    denom = max(1.0, run_max)
    pad = window - len(ring)
    for i, c in enumerate(ring):
        out[pad + i] = c / denom
    return out
