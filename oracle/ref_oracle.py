"""numpy restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.

Every function names the reference lines it restates (paths relative to
/root/reference/pkg/src/subnewton/).  Arithmetic is fp64 numpy/BLAS, the
same library stack the reference runs on, so on identical inputs the
results agree with the reference to rounding (pinned by tests/golden/).

Conventions (softmax.py:1-16, 62-74):
  * C classes, p features, K = C-1 weighted classes, d = K*p.
  * flat weights x are class-major: x[c*p + j] is feature j of class c;
    the matrix view is Wm = x.reshape((p, K), order="F"), Wm[j, c].
  * class C-1 is the reference class with implicit zero weights.
"""

import math

import numpy as np

__all__ = [
    "ROW_BLOCK", "CURVATURE_EPS", "VARIANTS",
    "CurvatureFailure", "ArmijoFailure",
    "stream_rng", "sample_size", "draw_index_set", "draw_samples",
    "weights_matrix", "row_terms", "data_loss", "loss", "data_grad", "grad",
    "hess_probs", "hess_apply", "class_probs", "predict", "accuracy",
    "cg", "armijo", "minimize", "newton_solve", "estimate_lipschitz",
    "synthetic_problem", "column_norms", "normalize_columns", "train_test_split",
]

ROW_BLOCK = 8192          # softmax.py:25 (BLOCK_ROWS)
CURVATURE_EPS = 1e-32     # cg.py:16
VARIANTS = {              # newton.py:26-30
    "full": (1.0, 1.0),
    "subsampled-100": (1.0, 0.05),
    "subsampled-20": (0.2, 0.05),
}
_U64 = (1 << 64) - 1      # rng.py:23


class CurvatureFailure(RuntimeError):
    """cg.py:78-83 (CurvatureError)."""


class ArmijoFailure(RuntimeError):
    """linesearch.py:54-57, 67-70 (LineSearchError)."""


# ----------------------------------------------------------------- rng / samples
def stream_rng(seed, *path):
    """rng.py:26-33: Philox keyed by SeedSequence([seed, *path]) (64-bit masked)."""
    key = [int(v) & _U64 for v in (seed, *path)]
    return np.random.Generator(np.random.Philox(seed=np.random.SeedSequence(key)))


def sample_size(fraction, n):
    """sampling.py:34-35 -- Python round() (half to even), floor of 1."""
    return max(1, int(round(fraction * n)))


def draw_index_set(gen, n, size, with_replacement):
    """sampling.py:38-45: sorted draw; the full sample is arange(n) in order."""
    if with_replacement:
        return np.sort(gen.integers(0, n, size=size))
    if size == n:
        return np.arange(n)
    return np.sort(gen.choice(n, size=size, replace=False))


def draw_samples(gradient_fraction, hessian_fraction, with_replacement, seed, n, iteration):
    """sampling.py:48-69: (S_g, S_H) from streams (seed, k, 0) and (seed, k, 1)."""
    if n < 1:
        raise ValueError("cannot sample from an empty dataset")
    s_g = draw_index_set(stream_rng(seed, iteration, 0), n,
                         sample_size(gradient_fraction, n), with_replacement)
    s_h = draw_index_set(stream_rng(seed, iteration, 1), n,
                         sample_size(hessian_fraction, n), with_replacement)
    return s_g, s_h


# ----------------------------------------------------------------- softmax pieces
def weights_matrix(x, p, C):
    """softmax.py:62-74: flat class-major x -> p-by-K matrix (Fortran view)."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != ((C - 1) * p,):
        raise ValueError(f"weight vector must have length {(C - 1) * p}, got {x.shape}")
    return x.reshape((p, C - 1), order="F")


def _row_blocks(n, rows=ROW_BLOCK):
    """softmax.py:102-104."""
    start = 0
    while start < n:
        stop = min(start + rows, n)
        yield start, stop
        start = stop


def row_terms(A, y, Wm, C):
    """softmax.py:85-99 for one block of rows.

    Returns (M, E, alpha, lin): M_i = max(0, max_c z_ic), E_ic = exp(z_ic - M_i),
    alpha_i = exp(-M_i) + sum_c E_ic, lin_i = z_{i,y_i} when y_i < C-1 else 0.
    """
    Z = A @ Wm
    K = C - 1
    M = np.maximum(Z.max(axis=1), 0.0) if K > 0 else np.zeros(len(y))
    E = np.exp(Z - M[:, None])
    alpha = np.exp(-M) + E.sum(axis=1)
    lin = np.zeros(len(y))
    own = np.flatnonzero(y < K)
    lin[own] = Z[own, y[own]]
    return M, E, alpha, lin


def data_loss(A, y, C, x):
    """softmax.py:125-135: sum_i (M_i + log alpha_i - lin_i), block order."""
    Wm = weights_matrix(x, A.shape[1], C)
    total = 0.0
    for a, b in _row_blocks(A.shape[0]):
        M, _, alpha, lin = row_terms(A[a:b], y[a:b], Wm, C)
        total += float((M + np.log(alpha) - lin).sum())
    return total


def loss(A, y, C, x, lam):
    """softmax.py:138-141: data loss + lam/2 ||x||^2."""
    x = np.asarray(x, dtype=np.float64)
    return data_loss(A, y, C, x) + 0.5 * lam * float(x @ x)


def data_grad(A, y, C, x):
    """softmax.py:144-163: vec_F( sum_blocks A_b^T (E/alpha - onehot) )."""
    p = A.shape[1]
    K = C - 1
    Wm = weights_matrix(x, p, C)
    G = np.zeros((p, K))
    for a, b in _row_blocks(A.shape[0]):
        yb = y[a:b]
        _, E, alpha, _ = row_terms(A[a:b], yb, Wm, C)
        R = E / alpha[:, None]
        own = np.flatnonzero(yb < K)
        R[own, yb[own]] -= 1.0
        G += A[a:b].T @ R
    return G.ravel(order="F")


def grad(A, y, C, x, lam, scale=1.0):
    """softmax.py:166-169 (scale = 1) and sampling.py:84-87 (scale = n/|S_g|)."""
    x = np.asarray(x, dtype=np.float64)
    return scale * data_grad(A, y, C, x) + lam * x


def hess_probs(A, y, C, x):
    """softmax.py:181-195: h_ic = E_ic / alpha_i on the rows of A (cached once)."""
    Wm = weights_matrix(x, A.shape[1], C)
    h = np.empty((A.shape[0], C - 1))
    for a, b in _row_blocks(A.shape[0]):
        _, E, alpha, _ = row_terms(A[a:b], y[a:b], Wm, C)
        h[a:b] = E / alpha[:, None]
    return h


def hess_apply(A, h, C, v, scale=1.0, lam=0.0):
    """softmax.py:197-210: scale * vec_F(A^T (V*h - h*rowsum(V*h))) + lam v, V = A Q."""
    v = np.asarray(v, dtype=np.float64)
    Q = weights_matrix(v, A.shape[1], C)
    acc = np.zeros(Q.shape)
    for a, b in _row_blocks(A.shape[0]):
        hb = h[a:b]
        VW = (A[a:b] @ Q) * hb
        U = VW - hb * VW.sum(axis=1)[:, None]
        acc += A[a:b].T @ U
    return scale * acc.ravel(order="F") + lam * v


def class_probs(A, y, C, x):
    """softmax.py:224-236: n-by-C probabilities, reference class last."""
    Wm = weights_matrix(x, A.shape[1], C)
    P = np.empty((A.shape[0], C))
    for a, b in _row_blocks(A.shape[0]):
        M, E, alpha, _ = row_terms(A[a:b], y[a:b], Wm, C)
        P[a:b, :-1] = E / alpha[:, None]
        P[a:b, -1] = np.exp(-M) / alpha
    return P


def predict(A, y, C, x):
    """softmax.py:239-240: argmax, ties to the lowest class index."""
    return np.argmax(class_probs(A, y, C, x), axis=1)


def accuracy(A, y, C, x):
    """softmax.py:243-247."""
    if A.shape[0] == 0:
        raise ValueError("accuracy is undefined on an empty dataset")
    return float(np.mean(predict(A, y, C, x) == y))


# ----------------------------------------------------------------- solvers
def cg(apply_H, g, theta=1e-4, max_iters=10):
    """cg.py:51-98: CG on H p = -g from p0 = 0 with best-residual tracking.

    Returns (p_best, r_best_norm, iterations, converged).
    """
    g = np.asarray(g, dtype=np.float64)
    gn = float(np.linalg.norm(g))
    if gn == 0.0:
        return np.zeros_like(g), 0.0, 0, True
    tol = theta * gn
    r = -g
    s = r.copy()
    p = np.zeros_like(g)
    best, best_norm = s.copy(), gn
    rr = float(r @ r)
    it, done = 0, False
    while it < max_iters:
        Hs = apply_H(s)
        it += 1
        sHs = float(s @ Hs)
        if sHs <= CURVATURE_EPS * float(s @ s):
            raise CurvatureFailure(f"non-positive curvature {sHs:.3e} at CG iteration {it}")
        a = rr / sHs
        p = p + a * s
        r = r - a * Hs
        rn = float(np.linalg.norm(r))
        if rn <= best_norm:
            best_norm, best = rn, p.copy()
        if rn <= tol:
            done = True
            break
        rr_new = float(r @ r)
        s = r + (rr_new / rr) * s
        rr = rr_new
    return best, best_norm, it, done


def armijo(f, f0, slope, beta=1e-4, rho=0.5, max_iters=50, alpha0=1.0):
    """linesearch.py:36-70: first alpha0*rho^i with f(alpha) <= f0 + alpha*beta*slope.

    Returns (alpha, evaluations); non-finite trials fail the test.
    """
    if not np.isfinite(f0):
        raise ArmijoFailure(f"objective at the current point is not finite: {f0}")
    if slope >= 0.0:
        raise ArmijoFailure(f"not a descent direction: p^T g = {slope:.3e} >= 0")
    alpha = alpha0
    for evals in range(1, max_iters + 2):
        trial = f(alpha)
        if np.isfinite(trial) and trial <= f0 + alpha * beta * slope:
            return alpha, evals
        alpha *= rho
    raise ArmijoFailure(f"no Armijo step after {max_iters + 1} evaluations")


def minimize(objective_fn, oracle_factory, x0, epsilon=1e-8, max_outer_iters=100,
             theta=1e-4, cg_max_iters=10, ls=None, metrics=None):
    """newton.py:60-112 -- the generic inexact Newton-CG loop.

    oracle_factory(k) returns (grad_fn, hess_apply_fn_factory) where
    hess_apply_fn_factory(x) returns v -> H v.
    Returns dict(records=[(k, f, train_acc, test_acc, alpha, cg_iters)], x, reason).
    """
    ls = dict(ls or {})
    x = np.array(x0, dtype=np.float64)
    metrics = metrics or (lambda _x: (math.nan, math.nan))
    f_cur = objective_fn(x)
    tr, te = metrics(x)
    records = [(0, f_cur, tr, te, 0.0, 0)]
    reason = "max-iters"
    for k in range(max_outer_iters):
        grad_fn, hess_factory = oracle_factory(k)
        g = grad_fn(x)
        if np.linalg.norm(g) < epsilon:
            reason = "gradient-converged"
            break
        p, _, iters, _ = cg(hess_factory(x), g, theta, cg_max_iters)
        slope = float(p @ g)
        try:
            alpha, _ = armijo(lambda a: objective_fn(x + a * p), f_cur, slope, **ls)
        except ArmijoFailure:
            reason = "line-search-failure"
            break
        x = x + alpha * p
        f_cur = objective_fn(x)
        tr, te = metrics(x)
        records.append((k + 1, f_cur, tr, te, alpha, iters))
    return {"records": records, "x": x, "reason": reason}


def newton_solve(A, y, C, lam, variant="subsampled-100", seed=0, epsilon=1e-8,
                 max_outer_iters=100, theta=1e-4, cg_max_iters=10, x0=None,
                 with_replacement=False, ls=None, test=None,
                 gradient_fraction=None, hessian_fraction=None):
    """newton.py:115-140 composed with sampling.py:72-96 (SubsampledOracle)."""
    n, p = A.shape
    f_g, f_h = VARIANTS[variant]
    if gradient_fraction is not None:
        f_g = gradient_fraction
    if hessian_fraction is not None:
        f_h = hessian_fraction
    x0 = np.zeros((C - 1) * p) if x0 is None else x0

    def factory(k):
        s_g, s_h = draw_samples(f_g, f_h, with_replacement, seed, n, k)
        full_g = len(s_g) == n and np.array_equal(s_g, np.arange(n))
        full_h = len(s_h) == n and np.array_equal(s_h, np.arange(n))
        Ag, yg = (A, y) if full_g else (A[s_g], y[s_g])
        Ah, yh = (A, y) if full_h else (A[s_h], y[s_h])
        sg, sh = n / len(s_g), n / len(s_h)

        def grad_fn(x):
            return grad(Ag, yg, C, x, lam, scale=sg)

        def hess_factory(x):
            h = hess_probs(Ah, yh, C, x)
            return lambda v: hess_apply(Ah, h, C, v, scale=sh, lam=lam)

        return grad_fn, hess_factory

    def metrics(x):
        te = accuracy(test[0], test[1], C, x) if test is not None else math.nan
        return accuracy(A, y, C, x), te

    return minimize(lambda x: loss(A, y, C, x, lam), factory, x0, epsilon,
                    max_outer_iters, theta, cg_max_iters, ls, metrics)


def estimate_lipschitz(A, y, C, iters=200, seed=0):
    """bench.py:116-138: power iteration on the lam=0 Hessian at x = 0."""
    p = A.shape[1]
    d = (C - 1) * p
    x0 = np.zeros(d)
    h = hess_probs(A, y, C, x0)
    v = stream_rng(seed, 4).standard_normal(d)
    v /= np.linalg.norm(v)
    rq = 0.0
    for _ in range(iters):
        w = hess_apply(A, h, C, v, 1.0, 0.0)
        rq = float(v @ w)
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 0.0
        v = w / nw
    return rq


# ----------------------------------------------------------------- data preparation
def column_norms(A):
    """dataset.py:103-107 (dense): sqrt of the column sums of squares."""
    return np.sqrt((np.asarray(A, dtype=np.float64) ** 2).sum(axis=0))


def normalize_columns(A):
    """dataset.py:314-324 + scale_columns :109-118: nonzero columns to unit norm."""
    norms = column_norms(A)
    scale = np.ones_like(norms)
    nz = norms > 0
    scale[nz] = 1.0 / norms[nz]
    return np.asarray(A, dtype=np.float64) * scale


def train_test_split(n, train_fraction, seed):
    """dataset.py:327-342: (train, test) sorted row indices from the SPLIT stream."""
    if not 0.0 < train_fraction < 1.0:
        raise ValueError(f"train_fraction must be in (0, 1), got {train_fraction}")
    if n < 2:
        raise ValueError(f"need at least 2 rows to split, got {n}")
    n_train = int(np.ceil(train_fraction * n))
    perm = stream_rng(seed, 2).permutation(n)  # rng.py:19 SPLIT_STREAM
    return np.sort(perm[:n_train]), np.sort(perm[n_train:])


# ----------------------------------------------------------------- synthetic data
def synthetic_problem(n, p, C, seed=0, normalize=True, ill_conditioned=False):
    """Synthetic dataset per SURVEY.md section 8(d).

    Features N(0,1) (as tests/helpers.py:26-32 random_dataset); columns scaled to
    unit norm as dataset.py:314-324 normalize_columns, or for the ill-conditioned
    TR config scaled by logspace(2, -4, p) (tests/test_acceptance.py:223-229).
    Labels uniform in [0, C).  Returns (A float64 n-by-p C-order, y int64).
    """
    gen = np.random.default_rng(seed)
    A = gen.standard_normal((n, p))
    y = gen.integers(0, C, size=n).astype(np.int64)
    if ill_conditioned:
        A *= np.logspace(2, -4, p)
    elif normalize:
        norms = np.sqrt((A ** 2).sum(axis=0))
        scale = np.ones_like(norms)
        nz = norms > 0
        scale[nz] = 1.0 / norms[nz]
        A *= scale
    return np.ascontiguousarray(A), y
