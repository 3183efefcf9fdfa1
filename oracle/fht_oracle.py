"""ORACLE for the Brady dyadic Fast Hough Transform (arXiv 1811.06378) -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import this module. The product path (`paper_1811_06378_b200`) never does, and this
module never imports the product path: they share no code. Everything here is plain numpy in
float64 / int64 (an optional float32 recursion exists only as a debugging aid).

Citations: ``P:n`` = /root/reference/PAPER.md line n (section given), ``S:n`` = SPEC.md line n.
Readings of ambiguous passages are numbered as in DESIGN.md "Readings" (R1..R23, which follow
SURVEY.md §8(c)'s ambiguity ledger).

Functions and what pins them (tests/test_oracle_pins.py):

* `dyadic_pattern` -- recursion of S:71 (R1). Pinned by SPEC worked examples S:74-76
  (tests/golden/spec_examples.json), the bit closed form, endpoint law, step law, exact
  diagonal and complement identity.
* `hough_direct` (tier 1) -- the plain definition: cell (s, x0) is the sum of the padded
  image along the cyclic dyadic pattern (P:52 parametrization, P:65-67 padding, P:76 mod(w+h)).
  Pinned by golden SPEC examples S:84-85, the s = 0 row == column sums (numpy sum), the
  s = n-1 row == wrapped diagonal sums (numpy trace), row conservation, black zone
  (P:81), single-pixel 'angle', rasterised-pattern peak == n.
* `hough_recursive` (tier 2) -- the paper's Fig. 6 block-doubling iteration,
  level by level. Pinned by equality with tier 1 on random images (every cell).
* `full_hough` -- P:89-103 flip-and-concatenate (R7-R9). Pinned by seam identities,
  row count 2(w+h)-3, attribution thresholds (S:248-250 golden).
* `angle_plan` / `transformed_image` / `angle_range` -- §4 shear + scale (P:124, P:132,
  P:144-152; R12-R17). Pinned by: identity plan [0,45] == QA exactly, [-45,0] == QB with
  rows reversed, row conservation, scale/shear laws for the plan scalars. `shear_offsets`
  (R13) by hand-derived goldens (tests/golden/plan_readings.json) and the property e_y - g y in
  (-1/2, 1/2] in exact rational arithmetic; `scale_colmap` (R14) by goldens and the nearest-
  neighbour property |(c + 1/2) alpha - (u + 1/2)| <= alpha/2 of the scale law with the
  floor/ceil(alpha) multiplicity law for dilations; `angle_of_row` (R19) by the endpoint slopes
  (row 0 = theta_min, row Hp - 1 = theta_max exactly, tan equally spaced) and a rasterised line.
* `fhtshift_amounts` / `fhtshift` -- §5 (R11). Pinned by permutation, contiguity of
  the meaningful run, width law w + s, P:160's quoted row-0 / last-row shifts, and
  exact centring of the all-ones run for every pad (R11's generic rule, not only pad = Hp).
* `pattern_on_original` / `cell_segment` -- §3.2 steps 1-2 and §3.3 attribution
  (P:111-113): a Hough cell back to its discrete pattern on the original image. Pinned by SPEC's
  worked cases (S:195-197, S:257-258 golden), the round trip (drawing the pixels and
  transforming gives the pixel count at that cell, a maximal cell) and the black-zone
  characterisation.
* `hough_peaks` -- top-k 3x3 local maxima of a Hough plane (R25 in DESIGN.md). Pinned
  by planted-peak examples, the cyclic column neighbourhood and the plateau rule.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

QA, QB, QC, QD = 0, 1, 2, 3
QUADRANT_NAMES = ("QA", "QB", "QC", "QD")
# (transposed?, sigma) per quadrant -- R4: QA (I,+) QB (I,-) QC (I^T,-) QD (I^T,+).
QUADRANT_FRAME = {QA: (False, +1), QB: (False, -1), QC: (True, -1), QD: (True, +1)}


def next_pow2(n: int) -> int:
    """R3: non-power-of-two heights are zero-padded to the next power of two."""
    if n < 1:
        raise ValueError("size must be >= 1")
    p = 1
    while p < n:
        p *= 2
    return p


def _is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


# ----------------------------------------------------------------------------------------
# Dyadic pattern ("discrete patterns of certain type [11]"; Fig. 6)
# ----------------------------------------------------------------------------------------
def dyadic_pattern(n: int, x0: int, t: int, W: int) -> list[int]:
    """Columns of the dyadic pattern of an n-row strip starting at x0 with total shift t.

    S:71 (R1): n = 1 -> [x0]; otherwise top half = pattern(n/2, x0, t//2) and bottom half =
    pattern(n/2, (x0 + ceil(t/2)) mod W, t//2).
    """
    if not _is_pow2(n):
        raise ValueError("n must be a power of two")
    if not (0 <= t < n):
        raise ValueError("shift t must satisfy 0 <= t < n")
    if not (0 <= x0 < W):
        raise ValueError("x0 must satisfy 0 <= x0 < W")
    if n == 1:
        return [x0]
    half = n // 2
    top = dyadic_pattern(half, x0, t // 2, W)
    bottom = dyadic_pattern(half, (x0 + (t + 1) // 2) % W, t // 2, W)
    return top + bottom


_PATTERN_CACHE: dict[int, np.ndarray] = {}


def pattern_offsets(n: int) -> np.ndarray:
    """D[t][y]: unwrapped offset of the pattern with shift t at row y (x0 = 0, no wrap).

    The same S:71 recursion as `dyadic_pattern`, evaluated for all t at once:
    D_n[t] = D_{n/2}[t>>1] ++ (ceil(t/2) + D_{n/2}[t>>1]).
    """
    if not _is_pow2(n):
        raise ValueError("n must be a power of two")
    if n in _PATTERN_CACHE:
        return _PATTERN_CACHE[n]
    D = np.zeros((1, 1), dtype=np.int64)
    m = 1
    while m < n:
        t = np.arange(2 * m)
        inner = D[t >> 1]                                  # [2m][m]
        D = np.concatenate([inner, inner + ((t + 1) // 2)[:, None]], axis=1)
        m *= 2
    D.setflags(write=False)
    _PATTERN_CACHE[n] = D
    return D


def pattern_deviation(n: int, t: int) -> float:
    """max |pattern(y) - t*y/(n-1)| over rows (ideal line through the endpoints)."""
    if n < 2:
        raise ValueError("n must be >= 2")
    cols = np.array(dyadic_pattern(n, 0, t, 4 * n))
    ideal = t * np.arange(n) / (n - 1)
    return float(np.max(np.abs(cols - ideal)))


# ----------------------------------------------------------------------------------------
# Quadrant frames (R2-R6, R22)
# ----------------------------------------------------------------------------------------
@dataclass
class Frame:
    """The strip a quadrant transform runs on: `rows` (Hp x W, zero padded) and sign sigma."""
    rows: np.ndarray   # [Hp][W] padded strip, int64 or float64
    sigma: int
    h: int             # content height (rows that may hold pixels)
    w: int             # content width
    Hp: int
    W: int


def _as_acc(img: np.ndarray) -> np.ndarray:
    if np.issubdtype(img.dtype, np.integer):
        return img.astype(np.int64)
    return img.astype(np.float64)


def quadrant_frame(img: np.ndarray, quadrant: int, pad: int | None = None,
                   square_to: tuple[int, int] | None = None) -> Frame:
    """Pad the (possibly transposed) image: Hp = next_pow2(rows), W = cols + pad (pad = Hp).

    P:52 -- mostly horizontal lines use the transposed image. P:65-67 -- the image is extended
    by an h x h zero block so the result is (w + h) x h. `square_to=(Hp, Wp)` is the full-mode
    padding of R9 (both dimensions padded to powers of two before the quadrants are taken).
    """
    a = _as_acc(np.asarray(img))
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError("image must be a non-empty 2-D array")
    if square_to is not None:
        Hp0, Wp0 = square_to
        b = np.zeros((Hp0, Wp0), dtype=a.dtype)
        b[: a.shape[0], : a.shape[1]] = a
        a = b
    transposed, sigma = QUADRANT_FRAME[quadrant]
    if transposed:
        a = a.T
    h, w = a.shape
    Hp = next_pow2(h)
    if pad is None:
        pad = Hp
    if pad < 0:
        raise ValueError("pad must be >= 0")
    W = w + pad
    rows = np.zeros((Hp, W), dtype=a.dtype)
    rows[:h, :w] = a
    return Frame(rows=rows, sigma=sigma, h=h, w=w, Hp=Hp, W=W)


# ----------------------------------------------------------------------------------------
# Tier 1: the plain definition
# ----------------------------------------------------------------------------------------
def hough_of_frame_direct(fr: Frame) -> np.ndarray:
    """H[s][x0] = sum_y rows[y][(x0 + sigma * D_{Hp,s}(y)) mod W]   (S:80 post)."""
    Hp, W = fr.Hp, fr.W
    D = pattern_offsets(Hp)
    x0 = np.arange(W)
    out = np.zeros((Hp, W), dtype=fr.rows.dtype)
    for s in range(Hp):
        acc = np.zeros(W, dtype=fr.rows.dtype)
        for y in range(Hp):
            acc += fr.rows[y][(x0 + fr.sigma * D[s][y]) % W]
        out[s] = acc
    return out


def hough_direct(img: np.ndarray, quadrant: int, pad: int | None = None) -> np.ndarray:
    return hough_of_frame_direct(quadrant_frame(img, quadrant, pad))


def hough_cells_direct(fr: Frame, cells) -> np.ndarray:
    """Tier 1 evaluated only at the listed (s, x0) cells (for sampled parity at full size)."""
    Hp, W = fr.Hp, fr.W
    out = np.zeros(len(cells), dtype=fr.rows.dtype)
    ys = np.arange(Hp)
    cache: dict[int, np.ndarray] = {}
    for k, (s, x0) in enumerate(cells):
        if s not in cache:
            cache[s] = np.array(dyadic_pattern(Hp, 0, int(s), 4 * Hp + 4))
        cols = (int(x0) + fr.sigma * cache[s]) % W
        out[k] = fr.rows[ys, cols].sum()
    return out


# ----------------------------------------------------------------------------------------
# Tier 2: Fig. 6 block-doubling recursion
# ----------------------------------------------------------------------------------------
def recursion_levels(F: np.ndarray, sigma: int, levels: int) -> np.ndarray:
    """`levels` iterations of the Fig. 6 block doubling on F[b][t][x] (blocks of
    size n = F.shape[1] rows, cyclic width W = F.shape[2]); level k merges blocks 2b, 2b+1:

        F_k[b][t](x) = F_{k-1}[2b][t>>1](x) + F_{k-1}[2b+1][t>>1]((x + sigma*ceil(t/2)) mod W)
    """
    for _ in range(levels):
        nb, size, W = F.shape[0] // 2, F.shape[1], F.shape[2]
        G = np.empty((nb, 2 * size, W), dtype=F.dtype)
        for b in range(nb):
            A, B = F[2 * b], F[2 * b + 1]
            for t in range(2 * size):
                c = (t + 1) // 2
                G[b, t] = A[t >> 1] + np.roll(B[t >> 1], -sigma * c)
        F = G
    return F


def hough_of_frame_recursive(fr: Frame, dtype=None) -> np.ndarray:
    """All log2(Hp) levels of `recursion_levels` starting from F_0[r][0](x) = rows[r][x].
    `dtype=np.float32` gives the float32 debugging run."""
    rows = fr.rows if dtype is None else fr.rows.astype(dtype)
    Hp, W = fr.Hp, fr.W
    F = rows.reshape(Hp, 1, W).copy()          # F[b][t][x], blocks of size 1
    return recursion_levels(F, fr.sigma, Hp.bit_length() - 1)[0]


def hough_recursive(img: np.ndarray, quadrant: int, pad: int | None = None, dtype=None) -> np.ndarray:
    return hough_of_frame_recursive(quadrant_frame(img, quadrant, pad), dtype=dtype)


# ----------------------------------------------------------------------------------------
# Full Hough image (R7-R9, R23)
# ----------------------------------------------------------------------------------------
def full_padding(h: int, w: int) -> tuple[int, int]:
    """R9: full mode pads h -> Hp and w -> Wp so all four quadrants have width Wp + Hp."""
    return next_pow2(h), next_pow2(w)


def full_quadrants(img: np.ndarray, tier: int = 2, dtype=None) -> list[np.ndarray]:
    """The four quadrant images [QA, QB, QC, QD] of the full transform (QUADS layout, unflipped)."""
    h, w = np.asarray(img).shape
    Hp, Wp = full_padding(h, w)
    outs = []
    for q in (QA, QB, QC, QD):
        fr = quadrant_frame(img, q, square_to=(Hp, Wp))
        outs.append(hough_of_frame_recursive(fr, dtype) if tier == 2 else hough_of_frame_direct(fr))
    return outs


def concat_rows(Hp: int, Wp: int) -> int:
    """the concatenated image has 2(w + h) - 3 rows."""
    return 2 * (Hp + Wp) - 3


def attribute_row(R: int, Hp: int, Wp: int) -> tuple[int, int]:
    """P:111-113 thresholds (R8: a shared row belongs to the earlier quadrant). Returns (q, s)."""
    if not (0 <= R < concat_rows(Hp, Wp)):
        raise ValueError("row out of range")
    if R < Hp:                                   # QA flipped
        return QA, Hp - 1 - R
    if R < 2 * Hp - 1:                           # QB
        return QB, R - (Hp - 1)
    if R < 2 * Hp - 2 + Wp:                      # QC flipped
        return QC, Wp - 1 - (R - (2 * Hp - 2))
    return QD, R - (2 * Hp + Wp - 3)             # QD


def full_concat(quads: list[np.ndarray], Hp: int, Wp: int) -> np.ndarray:
    """'[315;0] flipped; [0;45]; [45;90] flipped; [90;135]' joined on common edge rows."""
    W = quads[0].shape[1]
    out = np.zeros((concat_rows(Hp, Wp), W), dtype=quads[0].dtype)
    for R in range(out.shape[0]):
        q, s = attribute_row(R, Hp, Wp)
        out[R] = quads[q][s]
    return out


def full_hough(img: np.ndarray, layout: str = "quads", tier: int = 2):
    h, w = np.asarray(img).shape
    Hp, Wp = full_padding(h, w)
    quads = full_quadrants(img, tier=tier)
    if layout == "quads":
        return quads
    if layout == "concat":
        return full_concat(quads, Hp, Wp)
    raise ValueError(layout)


# ----------------------------------------------------------------------------------------
# §4 angle range (R12-R17)
# ----------------------------------------------------------------------------------------
_EPS = 1e-9


@dataclass
class AnglePlan:
    theta_min_deg: float
    theta_max_deg: float
    k_lo: float
    k_hi: float
    alpha: float
    h: int
    w: int
    Hp: int
    w_content: int     # w' = ceil(alpha * w)
    W: int             # W'
    g: float           # shear in transformed pixels per row: alpha * (-k_lo)
    rows: int = 0      # output rows: Hp (§4 plan) or S_max + 1 (pruned plan); 0 means Hp
    transposed: bool = False  # mostly-horizontal plan: built on the transposed image (h, w are its)


def shear_offsets(g: float, n: int) -> np.ndarray:
    """R13: e_y = floor(g*y + 0.5) in double, multiply then add (no fused multiply-add)."""
    y = np.arange(n, dtype=np.float64)
    return np.floor(g * y + 0.5).astype(np.int64)


def scale_colmap(alpha: float, w: int, w_content: int) -> np.ndarray:
    """R14: nearest neighbour: colmap[u] = min(w-1, floor((u + 0.5) / alpha))."""
    u = np.arange(w_content, dtype=np.float64)
    return np.minimum(w - 1, np.floor((u + 0.5) / alpha).astype(np.int64))


def angle_plan(h: int, w: int, theta_min_deg: float, theta_max_deg: float,
               k_lo: float | None = None, k_hi: float | None = None) -> AnglePlan:
    """Shear by k_lo then scale by alpha = 1/(k_hi - k_lo) maps slopes [k_lo, k_hi] onto QA's [0, 1].

    Scale law P:124: tan beta' = alpha * tan beta. Shear law P:132: tan -> tan + tan(shear).
    Composition P:144. theta is the inclination from vertical, tan theta = dx/dy (R12).
    `k_lo`/`k_hi` may be supplied (R16: parity feeds the library plan's scalars in).
    """
    if not (-90.0 < theta_min_deg < theta_max_deg < 90.0):
        raise ValueError("need -90 < theta_min < theta_max < 90")
    if k_lo is None:
        k_lo = math.tan(math.radians(theta_min_deg))
    if k_hi is None:
        k_hi = math.tan(math.radians(theta_max_deg))
    alpha = 1.0 / (k_hi - k_lo)
    if alpha * w < 1.0:
        raise ValueError("alpha * w < 1: image scales to nothing")
    w_content = int(math.ceil(alpha * w - _EPS))
    Hp = next_pow2(h)
    g = alpha * (-k_lo)
    e = shear_offsets(g, h)
    D = pattern_offsets(Hp)[:, :h]                       # [s][y], y < h only (rows >= h are empty)
    spread = (e[None, :] - D).max(axis=1) - (e[None, :] - D).min(axis=1)
    W = w_content + max(Hp, int(spread.max()) + 1)       # R17: no two unwrapped lines fold together
    return AnglePlan(theta_min_deg, theta_max_deg, k_lo, k_hi, alpha, h, w, Hp, w_content, W, g, Hp)


def angle_plan_pruned(h: int, w: int, theta_min_deg: float, theta_max_deg: float,
                      k_lo: float | None = None, k_hi: float | None = None) -> AnglePlan:
    """Shift-range-pruned plan: shear only (P:132 shear law; alpha = 1, so colmap is the identity
    and w' = w). The slopes [k_lo, k_hi] become slopes [0, k_hi - k_lo] of the sheared image, i.e. its QA
    rows s = (k - k_lo)(Hp - 1) (R19), so only rows s <= S_max = ceil((k_hi - k_lo)(Hp - 1)) are
    needed -- the paper's point that the restricted transform costs less. Needs k_hi - k_lo <= 1
    (the rows must fit QA); W' by R17 over the kept rows."""
    if not (-90.0 < theta_min_deg < theta_max_deg < 90.0):
        raise ValueError("need -90 < theta_min < theta_max < 90")
    if k_lo is None:
        k_lo = math.tan(math.radians(theta_min_deg))
    if k_hi is None:
        k_hi = math.tan(math.radians(theta_max_deg))
    if not k_hi - k_lo <= 1.0:
        raise ValueError("pruned plan needs k_hi - k_lo <= 1")
    Hp = next_pow2(h)
    rows = min(Hp, int(math.ceil((k_hi - k_lo) * (Hp - 1) - _EPS)) + 1)
    g = -k_lo
    e = shear_offsets(g, h)
    D = pattern_offsets(Hp)[:rows, :h]
    spread = (e[None, :] - D).max(axis=1) - (e[None, :] - D).min(axis=1)
    W = w + max(Hp, int(spread.max()) + 1)
    return AnglePlan(theta_min_deg, theta_max_deg, k_lo, k_hi, 1.0, h, w, Hp, w, W, g, rows)


def plan_rows(plan: AnglePlan) -> int:
    return plan.rows if plan.rows else plan.Hp


def angle_plan_horizontal(h: int, w: int, phi_min_deg: float, phi_max_deg: float, pruned: bool = False,
                          k_lo: float | None = None, k_hi: float | None = None) -> AnglePlan:
    """Mostly-horizontal lines (the transposed image serves the mostly-horizontal quadrants):
    the same plan built on I^T (h, w of the plan are w, h of the image), angles phi measured from the
    horizontal, tan phi = dy/dx."""
    make = angle_plan_pruned if pruned else angle_plan
    p = make(w, h, phi_min_deg, phi_max_deg, k_lo=k_lo, k_hi=k_hi)
    p.transposed = True
    return p


def _plan_image(img: np.ndarray, plan: AnglePlan) -> np.ndarray:
    return np.asarray(img).T if plan.transposed else np.asarray(img)


def transformed_image(img: np.ndarray, plan: AnglePlan) -> np.ndarray:
    """Materialise T (Hp x W'): T[y][x'] = I[y][colmap[(x' - e_y) mod W']] if that index < w'."""
    a = _as_acc(np.asarray(img))
    h, w = a.shape
    assert (h, w) == (plan.h, plan.w)
    colmap = scale_colmap(plan.alpha, w, plan.w_content)
    e = shear_offsets(plan.g, h)
    T = np.zeros((plan.Hp, plan.W), dtype=a.dtype)
    xs = np.arange(plan.W)
    for y in range(h):
        u = (xs - e[y]) % plan.W
        ok = u < plan.w_content
        T[y, ok] = a[y, colmap[u[ok]]]
    return T


def angle_range(img: np.ndarray, plan: AnglePlan, tier: int = 2) -> np.ndarray:
    """H_{+1}(T) with cyclic width W' -- the QA transform of the sheared and scaled image."""
    T = transformed_image(_plan_image(img, plan), plan)
    fr = Frame(rows=T, sigma=+1, h=plan.h, w=plan.W, Hp=plan.Hp, W=plan.W)
    H = hough_of_frame_recursive(fr) if tier == 2 else hough_of_frame_direct(fr)
    return H[: plan_rows(plan)]      # a pruned plan keeps rows s <= S_max of the same transform


def range_cells_direct(img: np.ndarray, plan: AnglePlan, cells) -> np.ndarray:
    """The §4 definition evaluated at listed (s, x0) cells without materialising T:
    sum_y T[y][(x0 + D_s(y)) mod W'] with T as in `transformed_image`."""
    a = _as_acc(_plan_image(img, plan))
    colmap = scale_colmap(plan.alpha, plan.w, plan.w_content)
    e = shear_offsets(plan.g, plan.h)
    ys = np.arange(plan.h)
    out = np.zeros(len(cells), dtype=a.dtype)
    D = pattern_offsets(plan.Hp)
    for k, (s, x0) in enumerate(cells):
        u = (int(x0) + D[int(s)][: plan.h] - e) % plan.W
        ok = u < plan.w_content
        out[k] = a[ys[ok], colmap[u[ok]]].sum()
    return out


def angle_of_row(s: int, plan: AnglePlan) -> float:
    """R19 (P:52 'shift = h tg(phi)'): row s holds patterns of endpoint slope s / (Hp - 1) in the
    transformed image (D_s(Hp - 1) = s); the scale law divides by alpha and the shear law
     adds k_lo back: slope k_lo + s / (alpha (Hp - 1)), returned as degrees (from vertical;
    from horizontal for a transposed plan)."""
    k = plan.k_lo + s / (plan.alpha * (plan.Hp - 1)) if plan.Hp > 1 else plan.k_lo
    return math.degrees(math.atan(k))


def range_support(plan: AnglePlan) -> tuple[np.ndarray, np.ndarray]:
    """(start_s, len_s): the unwrapped meaningful run of each output row (R11 generic rule)."""
    e = shear_offsets(plan.g, plan.h)
    D = pattern_offsets(plan.Hp)[: plan_rows(plan), : plan.h]
    v = e[None, :] - D
    start = v.min(axis=1)
    length = v.max(axis=1) - start + plan.w_content
    return start, length


# ----------------------------------------------------------------------------------------
# §5 fhtshift (R11)
# ----------------------------------------------------------------------------------------
def _ceil_half(v: int) -> int:
    return -((-v) // 2)


def fhtshift_amounts_quadrant(Hp: int, W: int, sigma: int, w_frame: int | None = None) -> np.ndarray:
    """Right-rotation k_s of row s by R11's generic rule k = ceil((W - len)/2) - start, so that the
    row's meaningful run lands centred (P:172 'concentrated around its center in a single zone').

    The run of row s is the cells a line of the w_frame-wide frame can reach (width law P:156,
    w + h tg(alpha) -> w_frame + s): signed x0 in [-s, w_frame) for sigma=+1 (start = -s), in
    [0, w_frame + s) for sigma=-1 (start = 0); len = w_frame + s. With pad = W - w_frame this is
    ceil((pad + s)/2) (sigma=+1) and ceil((pad - s)/2) (sigma=-1). For the paper's pad = Hp it is
    P:160's 'row zero will shift by h and the last row by h/2 ... rows are shifted by h - i/2',
    i counted on the flipped image, i = Hp - s (R11). `w_frame` defaults to W - Hp.
    """
    wf = W - Hp if w_frame is None else w_frame
    out = []
    for s in range(Hp):
        start = -s if sigma > 0 else 0
        length = wf + s
        out.append((_ceil_half(W - length) - start) % W)
    return np.array(out, dtype=np.int64)


def fhtshift_amounts_range(plan: AnglePlan) -> np.ndarray:
    """Generic rule (R11): k = ceil((W' - len)/2) - start, so the run is centred."""
    start, length = range_support(plan)
    return np.array([(_ceil_half(plan.W - int(L)) - int(st)) % plan.W for st, L in zip(start, length)],
                    dtype=np.int64)


def fhtshift_rows(hough: np.ndarray, k: np.ndarray) -> np.ndarray:
    """out[s][x] = in[s][(x - k_s) mod W] (cyclic right rotation of each row)."""
    out = np.empty_like(hough)
    for s in range(hough.shape[0]):
        out[s] = np.roll(hough[s], int(k[s]))
    return out


def fhtshift_quadrant(hough: np.ndarray, sigma: int, pad: int | None = None) -> np.ndarray:
    """fhtshift of one quadrant image [Hp][W]; `pad` = the frame's extension W - w_frame (None: Hp,
    the paper's h x h extension and every full-mode quadrant)."""
    Hp, W = hough.shape
    return fhtshift_rows(hough, fhtshift_amounts_quadrant(Hp, W, sigma, W - (Hp if pad is None else pad)))


def fhtshift_quads(quads: list[np.ndarray]) -> list[np.ndarray]:
    return [fhtshift_quadrant(q, QUADRANT_FRAME[i][1]) for i, q in enumerate(quads)]


def fhtshift_concat(full: np.ndarray, Hp: int, Wp: int) -> np.ndarray:
    """Row R of the concatenated image is rotated by its attributed quadrant's rule."""
    W = full.shape[1]
    k = np.zeros(full.shape[0], dtype=np.int64)
    for R in range(full.shape[0]):
        q, s = attribute_row(R, Hp, Wp)
        n = Hp if q in (QA, QB) else Wp
        k[R] = fhtshift_amounts_quadrant(n, W, QUADRANT_FRAME[q][1])[s]
    return fhtshift_rows(full, k)


def fhtshift_range(hough: np.ndarray, plan: AnglePlan) -> np.ndarray:
    return fhtshift_rows(hough, fhtshift_amounts_range(plan))


# ----------------------------------------------------------------------------------------
# §3.2 / §3.3: from a Hough cell back to the original image; peaks
# ----------------------------------------------------------------------------------------
def pattern_on_original(h: int, w: int, quadrant: int, s: int, x0: int, n: int, W: int) -> list[tuple[int, int]]:
    """Pixels (x, y) of the original h x w image on the pattern of cell (s, x0) of `quadrant`.

    P:71 step 1: the pattern of the padded frame, frame column (x0 + sigma * D_s(y)) for frame rows
    y < n (n = the frame's padded row count). P:73-75 step 2: columns mod W (case b: the pattern
    leaving the right side re-enters on the left) and only pixels inside the original frame (case a);
    none left means the black zone (case c). QC/QD frames are the transposed image:
    frame (row y, column x) is original pixel (x = y, y = x).
    """
    transposed, sigma = QUADRANT_FRAME[quadrant]
    fh, fw = (w, h) if transposed else (h, w)
    D = pattern_offsets(n)[s]
    pix = []
    for y in range(min(fh, n)):
        xf = (x0 + sigma * int(D[y])) % W
        if xf < fw:
            pix.append((y, xf) if transposed else (xf, y))
    return pix


def cell_segment(mode: str, h: int, w: int, row: int, col: int, quadrant: int = QA, layout: str = "quads"):
    """Cell (row, col) of a QUADRANT or FULL Hough plane -> (quadrant, s, pixels). FULL QUADS: plane
    `quadrant`, s = row; CONCAT: P:111-113 attribution (R8); padding as the transform's (R9)."""
    if mode == "quadrant":
        transposed = QUADRANT_FRAME[quadrant][0]
        n = next_pow2(w if transposed else h)
        W = (h if transposed else w) + n
        q, s = quadrant, row
    else:
        Hp, Wp = next_pow2(h), next_pow2(w)
        W = Hp + Wp
        q, s = (quadrant, row) if layout == "quads" else attribute_row(row, Hp, Wp)
        n = Wp if QUADRANT_FRAME[q][0] else Hp
    if s >= n:
        return q, s, []
    return q, s, pattern_on_original(h, w, q, s, col, n, W)


def hough_peaks(H: np.ndarray, k: int) -> list[tuple[float, int, int]]:
    """Top-k peaks of one Hough plane H[s][x0] (R25): a cell is a peak when it beats each of its up to
    8 neighbours -- columns cyclic (x0 is taken mod W), rows not -- where a beats b iff
    v(a) > v(b), or v(a) == v(b) and a comes first in row-major order (a plateau keeps its first
    cell). Peaks ordered by value descending, then row-major index ascending; at most k."""
    R, W = H.shape
    peaks = []
    for r in range(R):
        for c in range(W):
            v = H[r, c]
            ok = True
            for dr in (-1, 0, 1):
                rr = r + dr
                if rr < 0 or rr >= R:
                    continue
                for dc in (-1, 0, 1):
                    if dr == 0 and dc == 0:
                        continue
                    cc = (c + dc) % W
                    if rr == r and cc == c:
                        continue
                    u = H[rr, cc]
                    if u > v or (u == v and rr * W + cc < r * W + c):
                        ok = False
                        break
                if not ok:
                    break
            if ok:
                peaks.append((v, r, c))
    peaks.sort(key=lambda t: (-t[0], t[1] * W + t[2]))
    return peaks[:k]
