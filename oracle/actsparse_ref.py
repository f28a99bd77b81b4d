"""TEST INFRASTRUCTURE — numpy restatement of the reference algorithms on the
TEAL decode hot path (the checker, never the product).

Every function cites the reference file:line it restates (paths relative to
``/root/reference``; ``pkg/src/actsparse/`` omitted).  Arithmetic order and
dtypes follow the reference exactly where the reference is bit-defined
(masks, sparse GEMV accumulation order, histogram binning / inversion), so
these functions reproduce the reference's outputs bit-for-bit; this is pinned
by ``tests/test_oracle_golden.py`` against fixtures generated from the real
reference (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import math

import numpy as np

MATRIX_NAMES = ("q", "k", "v", "o", "gate", "up", "down")
TAPS = ("pre_attn", "attn_out", "pre_mlp", "mlp_inter")
MATRIX_TAP = {"q": "pre_attn", "k": "pre_attn", "v": "pre_attn", "o": "attn_out",
              "gate": "pre_mlp", "up": "pre_mlp", "down": "mlp_inter"}
RMSNORM_EPS = 1e-6          # model.py:36
DEFAULT_BIN_COUNT = 4096    # sparsifier.py:21
HI_STD_MULTIPLE = 8.0       # sparsifier.py:22
_CHILD_TAG = 0x9E3779B9     # tensor.py:27


# ---- thresholding (sparsifier.py:120-155) -----------------------------------

def sparsify(x, t):
    """sparsifier.py:120-125: where(|x| <= t, +0.0, x); t compared in fp32
    (NumPy weak-scalar promotion rounds t to nearest f32)."""
    if not t >= 0.0:
        raise ValueError(f"threshold must be non-negative, got {t}")
    a = np.asarray(x, dtype=np.float32)
    return np.where(np.abs(a) <= np.float32(t), np.float32(0.0), a)


def keep_mask(x, t):
    """Complement of the prune predicate of sparsify: !(|x| <= fl32(t))."""
    a = np.asarray(x, dtype=np.float32)
    return ~(np.abs(a) <= np.float32(t))


def realized_sparsity(x, t):
    """sparsifier.py:128-133."""
    a = np.asarray(x, dtype=np.float32)
    if a.size == 0:
        raise ValueError("realized sparsity of an empty vector is undefined")
    return float(np.count_nonzero(np.abs(a) <= np.float32(t))) / a.size


def sparsify_batched(xs, t):
    """sparsifier.py:136-155: shared column mask on mean_b |X[b, i]| <= t."""
    if not t >= 0.0:
        raise ValueError(f"threshold must be non-negative, got {t}")
    batch = np.asarray(xs, dtype=np.float32)
    mask = np.abs(batch).mean(axis=0) <= np.float32(t)
    out = batch.copy()
    out[:, mask] = np.float32(0.0)
    return out, mask


def pack_bits(keep):
    """keep (bool[m]) -> uint32 words, bit i%32 of word i//32 (GPU bitmask layout)."""
    keep = np.asarray(keep, dtype=bool).ravel()
    words = (keep.size + 31) // 32
    padded = np.zeros(words * 32, dtype=bool)
    padded[: keep.size] = keep
    bits = np.packbits(padded.reshape(-1, 32), axis=1, bitorder="little")
    return bits.view("<u4").ravel().astype(np.uint32)


# ---- GEMV (kernel.py:30-65, tensor.py:107-140) -------------------------------

def skip_gemv(x, w_in_major, t):
    """kernel.py:30-44 `_skip_gemv`: for i ascending, skip iff abs(x_i) <= t
    (fp64 compare of the f32 value against the Python float t), else
    y[:] += x_i * W[i, :] in fp32.  Returns (y, used).

    ``w_in_major`` is the [m, n] input-major (COL_MAJOR) storage."""
    x = np.asarray(x, dtype=np.float32)
    w = np.asarray(w_in_major, dtype=np.float32)
    m, n = w.shape
    y = np.zeros(n, dtype=np.float32)
    used = 0
    tt = float(t)
    for i in range(m):
        xi = x[i]
        if abs(float(xi)) <= tt:
            continue
        used += 1
        y += xi * w[i]
    return y, used


def gemv_dense(x, w_in_major):
    """tensor.py:107-127: y_j = sum_i x_i W[j, i], fp32, ascending i."""
    x = np.asarray(x, dtype=np.float32)
    w = np.asarray(w_in_major, dtype=np.float32)
    y = np.zeros(w.shape[1], dtype=np.float32)
    for i in range(w.shape[0]):
        y = y + x[i] * w[i]
    return y


def traffic_model(n, m, realized, bytes_per_element=4):
    """kernel.py:78-91 (weight bytes dense / sparse, activation bytes)."""
    if n < 1 or m < 1 or bytes_per_element <= 0:
        raise ValueError("dimensions and element size must be positive")
    if not 0.0 <= realized <= 1.0:
        raise ValueError(f"realized sparsity must lie in [0, 1], got {realized}")
    dense = n * m * bytes_per_element
    return dense, (1.0 - realized) * dense, m * bytes_per_element


def rel_err(y, ref):
    """kernel.py:116-120 `_rel_error`."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    denom = float(np.linalg.norm(ref))
    if denom == 0.0:
        return float(np.linalg.norm(y))
    return float(np.linalg.norm(y - ref)) / denom


# ---- histogram calibration (sparsifier.py:63-117) ----------------------------

def hist_record(counts, overflow, x, hi):
    """sparsifier.py:68-83: fp64 binning idx = floor(|x|/hi*bins), clip, |x|>hi
    -> overflow.  Returns updated (counts int64[bins], overflow int)."""
    bins = counts.size
    mags = np.abs(np.asarray(x, dtype=np.float64)).ravel()
    if np.isnan(mags).any():
        raise ValueError("cannot record NaN activations")
    over = mags > hi
    inr = mags[~over]
    counts = counts.copy()
    if inr.size:
        idx = np.floor(inr / hi * bins).astype(np.int64)
        idx = np.minimum(np.maximum(idx, 0), bins - 1)
        counts += np.bincount(idx, minlength=bins).astype(np.int64)
    return counts, overflow + int(over.sum())


def hist_threshold(counts, overflow, hi, p):
    """sparsifier.py:94-117: CDF inversion with in-bin linear interpolation."""
    bins = counts.size
    total = int(counts.sum()) + int(overflow)
    if not 0.0 <= p <= 1.0:
        raise ValueError(f"sparsity must lie in [0, 1], got {p}")
    if total < 1:
        raise ValueError("cannot estimate a threshold from an empty histogram")
    if p == 0.0:
        return 0.0
    if p == 1.0:
        return hi
    cdf = np.cumsum(counts) / total
    idx = int(np.searchsorted(cdf, p, side="left"))
    if idx >= bins:
        return hi
    lo_mass = float(cdf[idx - 1]) if idx > 0 else 0.0
    mass = float(cdf[idx]) - lo_mass
    width = hi / bins
    left = idx * width
    if mass <= 0.0:
        return left
    return left + (p - lo_mass) / mass * width


# ---- theory (theory.py:34-63) -------------------------------------------------

def gaussian_threshold(p, sigma_x=1.0):
    """theory.py:34-63: P(|Z| <= t) = p by bisection on erf to 1e-12."""
    if not 0.0 <= p <= 1.0:
        raise ValueError(f"sparsity must lie in [0, 1], got {p}")
    if p == 0.0:
        return 0.0
    if p == 1.0:
        return math.inf

    def mass(t):
        return 2.0 * (0.5 * (1.0 + math.erf(t / math.sqrt(2.0)))) - 1.0

    lo, hi = 0.0, 1.0
    while mass(hi) < p:
        hi *= 2.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if mass(mid) < p:
            lo = mid
        else:
            hi = mid
        if hi - lo <= 1e-12:
            break
    return sigma_x * 0.5 * (lo + hi)


# ---- seeded generation (tensor.py:146-171, model.py:106-123, 387-391) --------

def philox_generator(seed, counter):
    """tensor.py:164-167: Philox keyed by SeedSequence(seed, spawn_key=(counter,))."""
    ss = np.random.SeedSequence(entropy=int(seed) & 0xFFFF_FFFF_FFFF_FFFF, spawn_key=(int(counter),))
    return np.random.Generator(np.random.Philox(ss))


def child_seed(seed, index):
    """tensor.py:169-171."""
    ss = np.random.SeedSequence(entropy=int(seed) & 0xFFFF_FFFF_FFFF_FFFF, spawn_key=(_CHILD_TAG, int(index)))
    return int(ss.generate_state(1, np.uint64)[0])


def gen_block_weights(seed, d_model, heads, d_ff, counter=0):
    """model.py:106-123: weights W_name [n_out, d_in] ~ N(0, 1/d_in) drawn in the
    fixed order q,k,v,o,gate,up,down from one generator; unit norm scales."""
    g = philox_generator(seed, counter)
    shapes = {"q": (d_model, d_model), "k": (d_model, d_model), "v": (d_model, d_model),
              "o": (d_model, d_model), "gate": (d_ff, d_model), "up": (d_ff, d_model),
              "down": (d_model, d_ff)}
    out = {}
    for name in MATRIX_NAMES:
        n_out, d_in = shapes[name]
        std = np.float32(1.0 / math.sqrt(d_in))
        out[name] = g.standard_normal((n_out, d_in), dtype=np.float32) * std
    ones = np.ones(d_model, dtype=np.float32)
    return out, ones, ones.copy()


def gen_model_weights(seed, n_blocks, d_model, heads, d_ff):
    """model.py:387-391: block b uses RngStream(child(b))."""
    return [gen_block_weights(child_seed(seed, b), d_model, heads, d_ff) for b in range(n_blocks)]


# ---- block forward (model.py:126-198) ----------------------------------------

def rmsnorm(x, scale):
    """model.py:126-128."""
    ms = np.mean(x * x, axis=-1, keepdims=True)
    return x / np.sqrt(ms + np.float32(RMSNORM_EPS)) * scale


def silu(z):
    """model.py:131-132."""
    return z / (np.float32(1.0) + np.exp(-z))


def causal_attention(q, k, v, heads):
    """model.py:135-150 (MHA, no positional encoding)."""
    *lead, s, d = q.shape
    dh = d // heads

    def split(a):
        return np.swapaxes(a.reshape(*lead, s, heads, dh), -3, -2)

    sc = split(q) @ np.swapaxes(split(k), -1, -2)
    sc = sc / np.float32(math.sqrt(dh))
    sc = np.where(np.triu(np.ones((s, s), dtype=bool), k=1), np.float32(-np.inf), sc)
    sc = sc - sc.max(axis=-1, keepdims=True)
    e = np.exp(sc)
    p = e / e.sum(axis=-1, keepdims=True)
    return np.swapaxes(p @ split(v), -3, -2).reshape(*lead, s, d)


def block_forward(weights, rms_attn, rms_mlp, heads, X, thresholds=None, collect=None):
    """model.py:158-198 `_forward`: 7 masked projections at 4 taps."""
    x = np.asarray(X, dtype=np.float32)

    def gated(name, a):
        return a if thresholds is None else sparsify(a, thresholds[name])

    h = rmsnorm(x, rms_attn)
    if collect is not None:
        collect["pre_attn"] = h
    q = gated("q", h) @ weights["q"].T
    k = gated("k", h) @ weights["k"].T
    v = gated("v", h) @ weights["v"].T
    ctx = causal_attention(q, k, v, heads)
    if collect is not None:
        collect["attn_out"] = ctx
    y = x + gated("o", ctx) @ weights["o"].T
    hm = rmsnorm(y, rms_mlp)
    if collect is not None:
        collect["pre_mlp"] = hm
    inter = silu(gated("gate", hm) @ weights["gate"].T) * (gated("up", hm) @ weights["up"].T)
    if collect is not None:
        collect["mlp_inter"] = inter
    return y + gated("down", inter) @ weights["down"].T


def calibrate_block(weights, rms_attn, rms_mlp, heads, samples, bins=DEFAULT_BIN_COUNT):
    """model.py:268-294: per-tap histograms, hi = 8 * f32 std of the first sequence.
    Returns {tap: (counts, overflow, hi)}."""
    batch = np.stack([np.asarray(s, dtype=np.float32) for s in samples])
    taps = {}
    block_forward(weights, rms_attn, rms_mlp, heads, batch, collect=taps)
    out = {}
    for tap in TAPS:
        values = taps[tap]
        first_std = float(values[0].std())
        hi = HI_STD_MULTIPLE * first_std
        counts, ov = hist_record(np.zeros(bins, dtype=np.int64), 0, values, hi)
        out[tap] = (counts, ov, hi)
    return out


def resolve_thresholds(hists, levels):
    """model.py:253-265: threshold of each matrix from its tap histogram."""
    return {n: hist_threshold(*_cnt_ov_hi(hists[MATRIX_TAP[n]]), levels[n]) for n in MATRIX_NAMES}


def _cnt_ov_hi(h):
    counts, ov, hi = h
    return counts, ov, hi


# ---- greedy allocation (greedy.py:76-127) ------------------------------------

def greedy_trace(weights, rms_attn, rms_mlp, heads, hists, x_cal, alpha):
    """greedy.py:76-127 Algorithm 1; returns list of (P, levels, chosen, error)."""
    x = np.asarray(x_cal, dtype=np.float32)
    fp = {n: weights[n].size for n in MATRIX_NAMES}
    F = sum(fp.values())
    deltas = {n: alpha * F / fp[n] for n in MATRIX_NAMES}
    y_gt = block_forward(weights, rms_attn, rms_mlp, heads, x)
    levels = {n: 0.0 for n in MATRIX_NAMES}
    steps = [(0.0, dict(levels), None, 0.0)]
    cache = {}

    def thr(lv):
        out = {}
        for n in MATRIX_NAMES:
            key = (n, lv[n])
            if key not in cache:
                cache[key] = hist_threshold(*hists[MATRIX_TAP[n]], lv[n])
            out[n] = cache[key]
        return out

    P = 0.0
    while P < 1.0:
        best, best_lv, best_err = None, 0.0, math.inf
        for n in MATRIX_NAMES:
            if levels[n] >= 1.0:
                continue
            trial = min(levels[n] + deltas[n], 1.0)
            saved = levels[n]
            levels[n] = trial
            diff = y_gt - block_forward(weights, rms_attn, rms_mlp, heads, x, thr(levels))
            err = float(np.sqrt(np.sum(np.square(diff, dtype=np.float64))))
            levels[n] = saved
            if err < best_err:
                best, best_lv, best_err = n, trial, err
        levels[best] = best_lv
        P = sum(levels[n] * fp[n] for n in MATRIX_NAMES) / F
        steps.append((P, dict(levels), best, best_err))
    return steps
