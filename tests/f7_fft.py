"""F7: T_l X as a d-dimensional linear convolution computed by FFT (numpy) — a second,
independent way to get T_l X, used to pin the oracle's gather (test_oracle_pins.py) and to check the
device pencil at full size (test_gpu_parity.py). Test helper only; shares nothing with the CUDA path."""
import numpy as np


def fft_apply(grid, d, n, ell, X):
    """F7: (T_l x)[k] = (g * x)[k + e_l + n 1] — d-dim linear convolution by FFT (numpy),
    independent of the oracle's gather. X: (N, r). Returns (N, r)."""
    L = 2 * n + 2
    g = np.asarray(grid).reshape((L,) * d)
    size = 3 * n + 2
    shape = (size,) * d
    ax = list(range(d))
    Gf = np.fft.fftn(g, shape, axes=ax)
    out = np.empty_like(X)
    sl = []
    for i in range(d):
        off = n + (1 if i == ell - 1 else 0)
        sl.append(slice(off, off + n + 1))
    for r in range(X.shape[1]):
        x = X[:, r].reshape((n + 1,) * d)
        conv = np.fft.ifftn(Gf * np.fft.fftn(x, shape, axes=ax), axes=ax)
        out[:, r] = conv[tuple(sl)].reshape(-1)
    return out
