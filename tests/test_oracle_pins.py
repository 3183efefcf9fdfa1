"""Pins for the oracle (`oracle/fht_oracle.py`) against things other than itself.

Each test names what fixes the expected value: a golden value from SPEC.md / PAPER.md
(tests/golden/spec_examples.json), a closed form, a numpy library routine, an invariant
the paper states, or brute force on tiny inputs. CPU only.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import fht_oracle as O
from synth import random_image

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
QN = {"QA": O.QA, "QB": O.QB, "QC": O.QC, "QD": O.QD}


# ---------------------------------------------------------------- dyadic pattern
@pytest.mark.parametrize("ex", GOLDEN["dyadic_pattern"], ids=lambda e: e["cite"])
def test_pattern_golden(ex):
    assert O.dyadic_pattern(ex["n"], ex["x0"], ex["t"], ex["W"]) == ex["cols"]


def _closed_form(n, t, y):
    """D_{n,t}(y) = sum_q bit_{K-1-q}(y) * ceil((t>>q)/2), K = log2 n (an independent formula)."""
    K = n.bit_length() - 1
    return sum(((y >> (K - 1 - q)) & 1) * (((t >> q) + 1) // 2) for q in range(K))


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16, 32, 64, 128, 256])
def test_pattern_closed_form_and_laws(n):
    D = O.pattern_offsets(n)
    for t in range(n):
        cols = [_closed_form(n, t, y) for y in range(n)]
        assert list(D[t]) == cols
        assert D[t][0] == 0 and D[t][n - 1] == t                 # endpoint law S:90
        assert set(np.diff(D[t]).tolist()) <= {0, 1}              # step law S:91
        # complement identity: D_{n,n-1-t}(y) = y - D_{n,t}(y)
        assert (D[n - 1 - t] == np.arange(n) - D[t]).all()
    assert (D[n - 1] == np.arange(n)).all()                       # exact 45-degree diagonal
    if n <= 64:
        for t in range(n):
            assert O.dyadic_pattern(n, 0, t, 4 * n) == list(D[t])


def test_pattern_rejects():
    with pytest.raises(ValueError):
        O.dyadic_pattern(3, 0, 0, 8)
    with pytest.raises(ValueError):
        O.dyadic_pattern(4, 0, 4, 8)
    with pytest.raises(ValueError):
        O.dyadic_pattern(4, 8, 0, 8)


@pytest.mark.parametrize("ex", GOLDEN["pattern_deviation"], ids=lambda e: e["cite"])
def test_pattern_deviation_golden(ex):
    assert O.pattern_deviation(ex["n"], ex["t"]) == pytest.approx(ex["dev"], abs=1e-15)


def test_pattern_deviation_endpoints_exact():
    for n in (2, 4, 8, 16, 64, 256, 1024):
        assert O.pattern_deviation(n, 0) == 0.0
        assert O.pattern_deviation(n, n - 1) == 0.0


# ---------------------------------------------------------------- quadrant transform
@pytest.mark.parametrize("ex", GOLDEN["quadrant_qa"], ids=lambda e: e["cite"])
def test_quadrant_golden(ex):
    img = np.array(ex["image"], dtype=np.int64)
    for fn in (O.hough_direct, O.hough_recursive):
        assert fn(img, O.QA).tolist() == ex["hough"]


@pytest.mark.parametrize("ex", GOLDEN["single_pixel_support"], ids=lambda e: e["cite"])
def test_single_pixel_golden(ex):
    img = np.zeros((ex["h"], ex["w"]), dtype=np.int64)
    img[ex["pixel_y"], ex["pixel_x"]] = 1
    for fn in (O.hough_direct, O.hough_recursive):
        H = fn(img, O.QA)
        assert H.shape[1] == ex["W"]
        sup = sorted([int(x0), int(s)] for s, x0 in np.argwhere(H))
        assert sup == sorted(ex["support_x0_s"])
        assert H.sum() == 4


@pytest.mark.parametrize("ex", GOLDEN["pad_dims"], ids=lambda e: e["cite"])
def test_pad_dims_golden(ex):
    img = np.ones((ex["h"], ex["w"]), dtype=np.int64)
    fr = O.quadrant_frame(img, QN[ex["quadrant"]])
    assert (fr.Hp, fr.W) == (ex["Hp"], ex["W"])


SHAPES = [(1, 1), (2, 2), (3, 5), (4, 4), (5, 3), (7, 9), (8, 8), (16, 16), (9, 16), (16, 6)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("q", [0, 1, 2, 3])
def test_tier2_equals_tier1(shape, q):
    img = random_image(shape, "i32", seed=shape[0] * 100 + shape[1] * 7 + q)
    for pad in (None, 0, 3):
        assert (O.hough_direct(img, q, pad) == O.hough_recursive(img, q, pad)).all()
    f = random_image(shape, "f32", seed=q + 17).astype(np.float64)
    np.testing.assert_allclose(O.hough_direct(f, q), O.hough_recursive(f, q), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("shape", [(4, 4), (7, 9), (16, 16), (32, 20)])
@pytest.mark.parametrize("q", [0, 1, 2, 3])
def test_special_rows_library(shape, q):
    """s = 0 is the vertical projection (numpy sum); s = Hp-1 is the wrapped 45-degree
    diagonal sum (numpy trace over the horizontally tiled strip)."""
    img = random_image(shape, "i32", seed=11 + q)
    fr = O.quadrant_frame(img, q)
    H = O.hough_recursive(img, q)
    assert (H[0] == fr.rows.sum(axis=0)).all()
    tiled = np.concatenate([fr.rows, fr.rows, fr.rows], axis=1)   # [Hp][3W]
    if fr.sigma < 0:
        tiled = tiled[:, ::-1]
    diag = []
    for x0 in range(fr.W):
        if fr.sigma > 0:
            diag.append(np.trace(tiled, offset=x0))
        else:  # column x0 - y in the original == column (3W-1-(x0+W)) + y in the reversed copy
            diag.append(np.trace(tiled, offset=3 * fr.W - 1 - (x0 + fr.W)))
    assert (H[fr.Hp - 1] == np.array(diag)).all()


@pytest.mark.parametrize("q", [0, 1, 2, 3])
def test_row_conservation(q):
    """every row sums to the image total (each pattern takes one pixel per row)."""
    for shape in [(5, 7), (16, 16), (32, 8)]:
        img = random_image(shape, "i32", seed=q * 3 + shape[1])
        H = O.hough_recursive(img, q)
        assert (H.sum(axis=1) == img.sum()).all()


def test_black_zone():
    """a triangular area is zero for every input. QA: x0 in [w, W-s); QB: [w+s, W)."""
    for shape in [(8, 8), (16, 5), (5, 16)]:
        img = random_image(shape, "i32", seed=shape[1]) + 1
        for q in (O.QA, O.QB):
            fr = O.quadrant_frame(img, q)
            H = O.hough_recursive(img, q)
            for s in range(fr.Hp):
                zone = range(fr.w, fr.W - s) if q == O.QA else range(fr.w + s, fr.W)
                assert (H[s, list(zone)] == 0).all()
                # and cells outside it are not structurally zero for a positive image
                live = [x for x in range(fr.W) if x not in zone]
                if fr.h == fr.Hp:
                    assert (H[s, live] > 0).all()


@pytest.mark.parametrize("n,w", [(8, 8), (16, 16), (32, 24)])
def test_rasterised_pattern_peak(n, w):
    """North star: a dyadic segment of length n fully inside the image gives a peak of
    exactly n at its (shift, position), the unique maximum."""
    rng = np.random.default_rng(n * w)
    D = O.pattern_offsets(n)
    for _ in range(12):
        s = int(rng.integers(0, min(n, w)))
        q = int(rng.integers(0, 2))
        sigma = +1 if q == 0 else -1
        x0 = int(rng.integers(0, w - s)) if sigma > 0 else int(rng.integers(s, w))
        img = np.zeros((n, w), dtype=np.int64)
        img[np.arange(n), x0 + sigma * D[s]] = 1
        H = O.hough_recursive(img, q)
        assert H[s, x0] == n
        assert (H == n).sum() == 1


# ---------------------------------------------------------------- full image
@pytest.mark.parametrize("shape", [(2, 2), (4, 4), (8, 8), (16, 16), (4, 8), (3, 5), (16, 4), (5, 16)])
def test_full_seams_and_size(shape):
    """P:89 'concatenating the quadrants ... by their common edge rows' (integer images:
    the shared rows are identical), P:103 size 2(w+h)-3 (with the R9 padding)."""
    img = random_image(shape, "i32", seed=sum(shape))
    Hp, Wp = O.full_padding(*shape)
    qa, qb, qc, qd = O.full_hough(img, "quads")
    assert qa.shape == qb.shape == (Hp, Hp + Wp) and qc.shape == qd.shape == (Wp, Hp + Wp)
    assert (qa[0] == qb[0]).all()
    assert (qb[Hp - 1] == qc[Wp - 1]).all()
    assert (qc[0] == qd[0]).all()
    full = O.full_hough(img, "concat")
    assert full.shape == (2 * (Hp + Wp) - 3, Hp + Wp)


@pytest.mark.parametrize("ex", GOLDEN["full_rows"], ids=lambda e: e["cite"])
def test_full_rows_golden(ex):
    full = O.full_hough(np.zeros((ex["h"], ex["w"]), dtype=np.int64), "concat")
    assert full.shape == (ex["rows"], ex["cols"])
    assert not full.any()


@pytest.mark.parametrize("ex", GOLDEN["attribute_row"], ids=lambda e: e["cite"])
def test_attribute_row_golden(ex):
    q, s = O.attribute_row(ex["row"], ex["P"], ex["P"])
    assert (O.QUADRANT_NAMES[q], s) == (ex["quadrant"], ex["s"])


def test_attribute_row_thresholds_paper():
    """P:111-113 thresholds: shift < h -> QA; h <= shift < 2h-1 -> QB; 2h-1 <= shift < 2h+w-2 -> QC."""
    for P in (4, 8, 16):
        for R in range(4 * P - 3):
            q, _ = O.attribute_row(R, P, P)
            want = O.QA if R < P else O.QB if R < 2 * P - 1 else O.QC if R < 2 * P + P - 2 else O.QD
            assert q == want


@pytest.mark.parametrize("P", [8, 16, 32])
def test_single_pixel_angle_figure(P):
    """a point maps to two segments ('angle') meeting on the common row.

    One nonzero cell per concatenated row; rows [0, 2P-1) lie within pattern_deviation of
    x0 = xp + (R-(P-1)) yp/(P-1); rows [2P-2, 4P-3) within it of x0 = yp + (3P-3-R) xp/(P-1);
    both pass through (2P-2, xp+yp)."""
    rng = np.random.default_rng(P)
    dev = max(O.pattern_deviation(P, t) for t in range(P))
    for _ in range(10):
        xp, yp = (int(v) for v in rng.integers(0, P, size=2))
        img = np.zeros((P, P), dtype=np.int64)
        img[yp, xp] = 1
        full = O.full_hough(img, "concat")
        W = full.shape[1]
        assert ((full != 0).sum(axis=1) == 1).all()
        x = np.argmax(full, axis=1)
        # signed columns (R6): sigma=+1 quadrants map x0 >= w to x0 - W; sigma=-1 keep x0
        sig = np.array([O.QUADRANT_FRAME[O.attribute_row(R, P, P)[0]][1] for R in range(4 * P - 3)])
        xs = np.where((sig > 0) & (x >= P), x - W, x)
        for R in range(4 * P - 3):
            ideal = xp + (R - (P - 1)) * yp / (P - 1) if R <= 2 * P - 2 else yp + (3 * P - 3 - R) * xp / (P - 1)
            assert abs(xs[R] - ideal) <= dev + 1e-9
        assert xs[2 * P - 2] == xp + yp


# ---------------------------------------------------------------- angle range (§4)
def test_plan_c4_values():
    """SURVEY §8(a) a6 numbers for config 4, from the scale law and shear law."""
    p = O.angle_plan(4096, 4096, -15.0, 15.0)
    assert p.alpha == pytest.approx(1.0 / (2 * math.tan(math.radians(15))), rel=1e-15)
    assert p.alpha * (p.k_hi - p.k_lo) == pytest.approx(1.0, rel=1e-15)
    assert p.w_content == 7644 and p.W == 11740 and p.g == pytest.approx(0.5, rel=1e-12)


@pytest.mark.parametrize("shape", [(8, 8), (16, 11), (5, 7), (32, 32)])
def test_range_identity_is_qa(shape):
    """Plan [0, 45] (no shear, alpha = 1) is exactly the QA quadrant."""
    img = random_image(shape, "i32", seed=shape[0] + 5)
    p = O.angle_plan(*shape, 0.0, 45.0)
    assert p.W == O.quadrant_frame(img, O.QA).W
    assert (O.angle_range(img, p) == O.hough_recursive(img, O.QA)).all()


@pytest.mark.parametrize("shape", [(8, 8), (16, 11), (5, 7), (32, 32)])
def test_range_negative_is_qb_reversed(shape):
    """Plan [-45, 0] (shear by one column per row) is QB with rows reversed (complement identity)."""
    img = random_image(shape, "i32", seed=shape[1] + 9)
    p = O.angle_plan(*shape, -45.0, 0.0)
    qb = O.hough_recursive(img, O.QB)
    assert p.W == qb.shape[1]
    assert (O.angle_range(img, p) == qb[::-1]).all()


def test_range_conservation_and_tiers():
    img = random_image((16, 16), "i32", seed=3)
    for tmin, tmax in [(-15, 15), (5, 40), (-30, -2), (-60, 10)]:
        p = O.angle_plan(16, 16, tmin, tmax)
        T = O.transformed_image(img, p)
        R = O.angle_range(img, p)
        assert (R.sum(axis=1) == T.sum()).all()
        assert (R == O.angle_range(img, p, tier=1)).all()


def test_range_peak_location():
    """Approximate (R14 is parity unpinned vs the paper): a rasterised line of slope k in
    [k_lo, k_hi] peaks within 2 rows of alpha (k - k_lo)(Hp - 1)."""
    P = 64
    for tmin, tmax, k in [(-15, 15, 0.1), (-15, 15, -0.2), (10, 40, 0.5), (-40, -10, -0.4)]:
        img = np.zeros((P, P), dtype=np.int64)
        ys = np.arange(P)
        xs = np.floor(20 + k * ys + 0.5).astype(int) if k > 0 else np.floor(44 + k * ys + 0.5).astype(int)
        img[ys, xs] = 1
        p = O.angle_plan(P, P, tmin, tmax)
        R = O.angle_range(img, p)
        s_peak = np.unravel_index(np.argmax(R), R.shape)[0]
        assert abs(s_peak - p.alpha * (k - p.k_lo) * (P - 1)) <= 2.0


# ---------------------------------------------------------------- shift-range-pruned plan (f2)
@pytest.mark.parametrize("shape", [(8, 8), (16, 11), (5, 7), (32, 32), (64, 40)])
@pytest.mark.parametrize("tmax", [10.0, 30.0, 45.0])
def test_pruned_zero_shear_is_qa_rows(shape, tmax):
    """theta in [0, tmax] needs no shear (k_lo = 0): the pruned transform is exactly the first
    ceil(tan(tmax)(Hp - 1)) + 1 rows of the QA quadrant (SURVEY §8(f) f2 pin; R19 row -> slope)."""
    img = random_image(shape, "i32", seed=shape[0] * 7 + int(tmax))
    p = O.angle_plan_pruned(*shape, 0.0, tmax)
    Hp = O.next_pow2(shape[0])
    assert p.rows == min(Hp, math.ceil(math.tan(math.radians(tmax)) * (Hp - 1) - 1e-9) + 1)
    qa = O.hough_recursive(img, O.QA)
    assert p.W == qa.shape[1]
    assert (O.angle_range(img, p) == qa[: p.rows]).all()


def test_pruned_conservation_and_tiers():
    """alpha = 1: T holds every pixel once, so every kept row sums to the image total; tier 1
    (direct pattern sums) equals tier 2 on every kept cell."""
    img = random_image((32, 24), "i32", seed=11)
    for tmin, tmax in [(-15, 15), (5, 40), (-30, -2), (-26, 18)]:
        p = O.angle_plan_pruned(32, 24, tmin, tmax)
        R = O.angle_range(img, p)
        assert R.shape == (p.rows, p.W)
        assert (R.sum(axis=1) == img.sum()).all()
        assert (R == O.angle_range(img, p, tier=1)).all()
        start, length = O.range_support(p)
        assert len(start) == p.rows and (length <= p.W).all()


def test_pruned_peak_location():
    """A digital line of slope k in [k_lo, k_hi] peaks at row (k - k_lo)(Hp - 1) of the sheared frame
    (within 2 rows: the shear is rounded per row)."""
    P = 64
    for tmin, tmax, k in [(-15, 15, 0.1), (-15, 15, -0.2), (10, 40, 0.5), (-40, -10, -0.4)]:
        img = np.zeros((P, P), dtype=np.int64)
        ys = np.arange(P)
        xs = np.floor(20 + k * ys + 0.5).astype(int) if k > 0 else np.floor(44 + k * ys + 0.5).astype(int)
        img[ys, xs] = 1
        p = O.angle_plan_pruned(P, P, tmin, tmax)
        R = O.angle_range(img, p)
        s_peak = np.unravel_index(np.argmax(R), R.shape)[0]
        assert abs(s_peak - (k - p.k_lo) * (P - 1)) <= 2.0
        assert R.max() >= P // 2          # the line's pixels concentrate in one cell (not exact: DDA != dyadic)


@pytest.mark.parametrize("shape", [(8, 8), (16, 11), (5, 7), (32, 20)])
def test_horizontal_plan_is_qd_qc(shape):
    """Mostly-horizontal plans (f4): [0, 45] from the horizontal is exactly QD (I^T, +), and
    [-45, 0] is QC (I^T, -) with rows reversed -- the transposed counterparts of the QA / QB pins."""
    img = random_image(shape, "i32", seed=shape[0] * 11 + shape[1])
    p = O.angle_plan_horizontal(*shape, 0.0, 45.0)
    qd = O.hough_recursive(img, O.QD)
    assert (p.h, p.w) == (shape[1], shape[0]) and p.W == qd.shape[1]
    assert (O.angle_range(img, p) == qd).all()
    q = O.angle_plan_horizontal(*shape, -45.0, 0.0)
    qc = O.hough_recursive(img, O.QC)
    assert (O.angle_range(img, q) == qc[::-1]).all()


def test_range_support_no_fold():
    """R17: with W' chosen by the rule, each row's unwrapped support fits in W' columns."""
    for tmin, tmax in [(-15, 15), (5, 40), (-80, 80), (1, 2)]:
        p = O.angle_plan(32, 24, tmin, tmax)
        start, length = O.range_support(p)
        assert (length <= p.W).all()


# ---------------------------------------------------------------- fhtshift (§5)
@pytest.mark.parametrize("ex", GOLDEN["fhtshift_qa_row_shift"], ids=lambda e: e["cite"])
def test_fhtshift_golden(ex):
    k = O.fhtshift_amounts_quadrant(ex["Hp"], 2 * ex["Hp"], +1)
    assert k[ex["s"]] == ex["k"]


@pytest.mark.parametrize("P", [4, 8, 16, 32])
def test_fhtshift_contiguous_centred(P):
    """P:156 width law w + h tg(alpha) -> w + s, P:172 'concentrated around its center ...
    a single zone without any gaps' -> one run, centred within half a column."""
    img = np.ones((P, P), dtype=np.int64)
    quads = O.full_hough(img, "quads")
    for q, H in enumerate(quads):
        S = O.fhtshift_quadrant(H, O.QUADRANT_FRAME[q][1])
        W = S.shape[1]
        for s in range(P):
            nz = np.flatnonzero(S[s])
            assert len(nz) == P + s and nz[-1] - nz[0] + 1 == len(nz)
            centre = (nz[0] + nz[-1] + 1) / 2
            assert abs(centre - W / 2) <= 0.5
            assert sorted(S[s].tolist()) == sorted(H[s].tolist())      # permutation


def test_fhtshift_permutation_random():
    img = random_image((16, 12), "i32", seed=5)
    full = O.full_hough(img, "concat")
    S = O.fhtshift_concat(full, 16, 16)
    for R in range(full.shape[0]):
        assert sorted(S[R].tolist()) == sorted(full[R].tolist())


def test_fhtshift_concat_contiguous():
    for P in (4, 8):
        full = O.full_hough(np.ones((P, P), dtype=np.int64), "concat")
        S = O.fhtshift_concat(full, P, P)
        for R in range(S.shape[0]):
            nz = np.flatnonzero(S[R])
            assert nz[-1] - nz[0] + 1 == len(nz)


def test_fhtshift_range_contiguous():
    for shape, tmin, tmax in [((16, 16), -15, 15), ((32, 20), 5, 40), ((16, 16), -45, 0)]:
        img = np.ones(shape, dtype=np.int64)
        p = O.angle_plan(*shape, tmin, tmax)
        R = O.angle_range(img, p)
        S = O.fhtshift_range(R, p)
        start, length = O.range_support(p)
        for s in range(p.Hp):
            nz = np.flatnonzero(S[s])
            assert nz[-1] - nz[0] + 1 == len(nz) == length[s]
            assert abs((nz[0] + nz[-1] + 1) / 2 - p.W / 2) <= 0.5


def test_float32_recursion_close_to_f64():
    """Debug aid (R21 tolerance): the float32 recursion is within 1e-3 + 1e-5|x| of f64."""
    img = random_image((64, 64), "f32", seed=1)
    a = O.hough_recursive(img, O.QA)
    b = O.hough_recursive(img, O.QA, dtype=np.float32)
    assert np.all(np.abs(a - b) <= 1e-3 + 1e-5 * np.abs(a))


def test_range_cells_direct_equals_materialised():
    img = random_image((24, 20), "i32", seed=8)
    for tmin, tmax in [(-15, 15), (5, 40), (-60, 10)]:
        p = O.angle_plan(24, 20, tmin, tmax)
        R = O.angle_range(img, p)
        cells = [(s, x) for s in range(p.Hp) for x in range(0, p.W, 3)]
        got = O.range_cells_direct(img, p, cells)
        assert (got == np.array([R[s, x] for s, x in cells])).all()


def test_cells_direct_equals_full():
    img = random_image((20, 13), "i32", seed=9)
    for q in range(4):
        fr = O.quadrant_frame(img, q)
        H = O.hough_of_frame_direct(fr)
        cells = [(s, x) for s in range(fr.Hp) for x in range(fr.W)]
        assert (O.hough_cells_direct(fr, cells) == H.ravel()).all()


# ---------------------------------------------------------------- §3.2 / §3.3 recovery, peaks (f3)
@pytest.mark.parametrize("ex", GOLDEN["pattern_on_original"], ids=lambda e: e["cite"])
def test_pattern_on_original_golden(ex):
    q = O.QUADRANT_NAMES.index(ex["quadrant"])
    n = O.next_pow2(ex["h"])
    pix = O.pattern_on_original(ex["h"], ex["w"], q, ex["s"], ex["x0"], n, ex["w"] + n)
    assert [list(p) for p in pix] == ex["pixels"]


@pytest.mark.parametrize("ex", GOLDEN["concat_cell_segment"], ids=lambda e: e["cite"])
def test_concat_cell_segment_golden(ex):
    q, s, pix = O.cell_segment("full", ex["h"], ex["w"], ex["row"], ex["col"], layout="concat")
    assert (O.QUADRANT_NAMES[q], s) == (ex["quadrant"], ex["s"])
    assert [list(p) for p in pix] == ex["pixels"]


def test_segment_round_trip():
    """drawing a recovered pattern into a blank image and transforming gives its pixel count at
    that cell, and no cell exceeds it (the tier-2 recursion does not use the pattern table)."""
    rng = np.random.default_rng(8)
    for _ in range(60):
        h, w = int(rng.integers(1, 17)), int(rng.integers(1, 17))
        q = int(rng.integers(0, 4))
        tr = O.QUADRANT_FRAME[q][0]
        n = O.next_pow2(w if tr else h)
        W = (h if tr else w) + n
        s, x0 = int(rng.integers(0, n)), int(rng.integers(0, W))
        pix = O.pattern_on_original(h, w, q, s, x0, n, W)
        if not pix:
            continue
        img = np.zeros((h, w), dtype=np.int64)
        for x, y in pix:
            img[y, x] = 1
        H = O.hough_recursive(img, q)
        assert H[s, x0] == len(pix) == H.max()


def test_black_zone_characterisation():
    """for QA (h a power of two) the pattern misses the image exactly when x0 >= w and
    x0 + s < W; for h < Hp the pattern ends at row h - 1, so s becomes its offset there, D_s(h - 1)."""
    for h, w in [(4, 4), (8, 5), (16, 16), (5, 12), (3, 7)]:
        n = O.next_pow2(h)
        W = w + n
        for s in range(n):
            reach = s if h == n else int(O.pattern_offsets(n)[s][h - 1])
            for x0 in range(W):
                empty = not O.pattern_on_original(h, w, O.QA, s, x0, n, W)
                assert empty == (x0 >= w and x0 + reach < W)


def test_full_cell_segment_quads_matches_quadrant():
    """FULL/QUADS recovery equals the quadrant's own recovery when the image is already square."""
    for q in range(4):
        for row, col in [(0, 0), (3, 5), (7, 15), (5, 9)]:
            _, _, a = O.cell_segment("full", 8, 8, row, col, quadrant=q)
            _, _, b = O.cell_segment("quadrant", 8, 8, row, col, quadrant=q)
            assert a == b


def test_hough_peaks_planted():
    """R25 rule on a planted plane: cyclic columns ((0,7) neighbours (0,0)), ties to the earlier cell,
    order by value then row-major index."""
    H = np.zeros((4, 8), dtype=np.int64)
    H[1, 2], H[2, 6], H[0, 7], H[0, 0] = 5, 7, 3, 3
    assert O.hough_peaks(H, 3) == [(7, 2, 6), (5, 1, 2), (3, 0, 0)]
    P = np.array([[1, 4, 4, 4, 1, 0], [0, 0, 0, 0, 0, 0]], dtype=np.int64)    # plateau: first cell only
    assert O.hough_peaks(P, 2) == [(4, 0, 1)]                                # zeros all lose to an earlier neighbour
    F = np.array([[0.5, -1.0, 0.25], [0.5, 2.0, -3.0]], dtype=np.float64)
    assert O.hough_peaks(F, 5) == [(2.0, 1, 1)]


# ---------------------------------------------------------------- round 2: the open readings pinned
PLAN_GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "plan_readings.json")))


@pytest.mark.parametrize("ex", PLAN_GOLDEN["shear_offsets"], ids=lambda e: str(e["g"]))
def test_shear_offsets_golden(ex):
    """R13: hand-derived shear offsets, ties rounding up."""
    assert O.shear_offsets(ex["g"], len(ex["e"])).tolist() == ex["e"]


@pytest.mark.parametrize("g", [0.5, -0.5, 0.25, 1.0 / 3.0, -0.7, 2.5, 0.0, 1.8660254037844388,
                               0.26794919243112275, -11.430052302761343])
def test_shear_offsets_nearest_ties_up(g):
    """R13 as a property: e_y is the integer nearest g*y with ties up, i.e. e_y - g*y in (-1/2, 1/2]
    (exact rational arithmetic on the double g). A floor shear (e - gy in (-1, 0]) or round-half-down
    (e - gy = -1/2 at a tie) fails."""
    from fractions import Fraction
    e = O.shear_offsets(g, 3000)
    G = Fraction(g)
    for y in range(3000):
        d = Fraction(int(e[y])) - G * y
        assert Fraction(-1, 2) < d <= Fraction(1, 2), (g, y, d)


@pytest.mark.parametrize("ex", PLAN_GOLDEN["scale_colmap"], ids=lambda e: str(e["alpha"]))
def test_scale_colmap_golden(ex):
    """R14 (P:124 scale law): hand-derived nearest-neighbour maps."""
    wc = math.ceil(ex["alpha"] * ex["w"] - 1e-9)
    assert O.scale_colmap(ex["alpha"], ex["w"], wc).tolist() == ex["colmap"]


@pytest.mark.parametrize("alpha", [1.8660254037844388, 2.0, 3.3, 1.0, 1.25, 0.7, 0.5, 0.25, 5.0])
@pytest.mark.parametrize("w", [7, 64, 100, 4096])
def test_scale_colmap_nearest_neighbour(alpha, w):
    """R14 as properties of nearest-neighbour resampling under the scale law x' = alpha x:
    transformed column u (centre u + 1/2) takes the source column c whose scaled centre (c + 1/2) alpha
    is nearest, |(c + 1/2) alpha - (u + 1/2)| <= alpha / 2 (clamped to w - 1 only past the right edge);
    for alpha >= 1 (a dilation) the map is onto and every interior source column is taken floor(alpha)
    or ceil(alpha) times. A corner-aligned map floor(u / alpha + 1/2) fails the first property."""
    wc = math.ceil(alpha * w - 1e-9)
    cm = O.scale_colmap(alpha, w, wc)
    assert len(cm) == wc and cm.min() >= 0 and cm.max() <= w - 1
    assert (np.diff(cm) >= 0).all()
    for u in range(wc):
        c = int(cm[u])
        if (u + 0.5) / alpha >= w:                      # past the last source centre band: clamped
            assert c == w - 1
            continue
        assert abs((c + 0.5) * alpha - (u + 0.5)) <= alpha / 2 + 1e-12, (u, c)
    if alpha >= 1.0:
        counts = np.bincount(cm, minlength=w)
        assert (counts >= 1).all()
        inner = counts[1:-1]
        assert ((inner == math.floor(alpha)) | (inner == math.ceil(alpha))).all()


@pytest.mark.parametrize("shape,tmin,tmax", [((64, 64), -15, 15), ((32, 40), 5, 40), ((128, 16), -60, 10),
                                             ((16, 16), -80, 80), ((256, 100), 1, 2)])
def test_angle_of_row_endpoints(shape, tmin, tmax):
    """R19 (P:52 'shift = h tg(phi)'): row s of the §4 frame holds patterns whose endpoint slope is
    s / (Hp - 1) (D_s(0) = 0, D_s(Hp - 1) = s) in the transformed image; undoing the scale law
     and shear law gives the image slope. So row 0 is theta_min, row Hp - 1 is theta_max
    exactly, and tan(angle) is equally spaced in s. A formula without the scale (alpha) or in radians
    fails the far endpoint."""
    p = O.angle_plan(*shape, tmin, tmax)
    a = np.array([O.angle_of_row(s, p) for s in range(p.Hp)])
    assert a[0] == pytest.approx(tmin, abs=1e-9) and a[-1] == pytest.approx(tmax, abs=1e-9)
    t = np.tan(np.radians(a))
    assert np.allclose(np.diff(t), (t[-1] - t[0]) / (p.Hp - 1), rtol=1e-9, atol=1e-12)
    assert (np.diff(a) > 0).all()
    # pruned plan: shear only (alpha = 1), row S_max is the first row at or past theta_max
    if math.tan(math.radians(tmax)) - math.tan(math.radians(tmin)) <= 1.0:
        q = O.angle_plan_pruned(*shape, tmin, tmax)
        assert O.angle_of_row(0, q) == pytest.approx(tmin, abs=1e-9)
        assert O.angle_of_row(q.rows - 1, q) >= tmax - 1e-9
        if q.rows >= 2:
            assert O.angle_of_row(q.rows - 2, q) < tmax


def test_angle_of_row_peak():
    """A rasterised line of known inclination peaks at a row whose angle_of_row is within 2 rows'
    worth of the line's angle (the shear and the digital line are rounded per row)."""
    P = 128
    for tmin, tmax, deg in [(-15, 15, 6.0), (-15, 15, -9.0), (10, 40, 25.0), (-40, -10, -20.0)]:
        k = math.tan(math.radians(deg))
        img = np.zeros((P, P), dtype=np.int64)
        ys = np.arange(P)
        xs = np.floor((30 if k > 0 else 90) + k * ys + 0.5).astype(int)
        img[ys, xs] = 1
        p = O.angle_plan(P, P, tmin, tmax)
        s_peak = int(np.unravel_index(np.argmax(O.angle_range(img, p)), (p.Hp, p.W))[0])
        dk = 2.0 / (p.alpha * (p.Hp - 1))           # slope step of 2 rows
        assert abs(math.tan(math.radians(O.angle_of_row(s_peak, p))) - k) <= dk


@pytest.mark.parametrize("P,w", [(8, 8), (16, 16), (16, 5), (8, 20)])
@pytest.mark.parametrize("q", [0, 1, 2, 3])
def test_fhtshift_centred_any_pad(P, w, q):
    """R11's generic rule for every pad (P:156 width law w + s, P:172 'concentrated around its center in
    a single zone'): for an all-ones P x w frame (h = Hp) and any pad >= s, row s's meaningful run of
    w_frame + s cells lands exactly at [ceil((W - len)/2), ...) -- centred, one zone. A shift taken from
    Hp instead of the pad (off by (pad - Hp)/2) fails."""
    shape = (P, w) if q < 2 else (w, P)                   # the frame is P rows x w columns
    img = np.ones(shape, dtype=np.int64)
    sigma = O.QUADRANT_FRAME[q][1]
    for pad in sorted({P - 1, P, P + 1, P + 7, 2 * P + 3, 40}):
        H = O.hough_recursive(img, q, pad)
        W = w + pad
        assert H.shape == (P, W)
        S = O.fhtshift_quadrant(H, sigma, pad)
        for s in range(P):
            assert sorted(S[s].tolist()) == sorted(H[s].tolist())      # a rotation of the row
            if s > pad:
                continue                                               # the run wraps onto itself
            L = w + s
            nz = np.flatnonzero(S[s])
            assert len(nz) == L and nz[0] == -((L - W) // 2) and nz[-1] == nz[0] + L - 1, (pad, s)
