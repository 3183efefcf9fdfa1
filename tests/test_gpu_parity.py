"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded inputs.

Bar: integer input -> bit-exact int32; float32 input -> |gpu - o64| <=
ATOL + RTOL |o64| with RTOL = 1e-5, ATOL = 1e-3 (north_star; R21). fhtshift is a bit copy
and is compared exactly against the oracle's rotation of the GPU's own unshifted output.
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-3


@pytest.fixture(scope="module")
def fht():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1811_06378_b200 as F
    return F


@pytest.fixture(scope="module")
def O():
    from oracle import fht_oracle
    return fht_oracle


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(got, want, integer):
    got = np.asarray(got)
    if integer:
        assert got.dtype == np.int32
        assert np.array_equal(got.astype(np.int64), want), f"max |diff| {np.abs(got.astype(np.int64) - want).max()}"
    else:
        assert got.dtype == np.float32
        err = np.abs(got.astype(np.float64) - want)
        bad = err > ATOL + RTOL * np.abs(want)
        assert not bad.any(), f"{bad.sum()} cells out of tolerance, max err {err.max()}"


SHAPES = [(1, 1), (2, 2), (3, 5), (5, 3), (7, 9), (16, 16), (33, 17), (64, 64), (100, 37), (129, 200), (256, 256)]


@pytest.mark.parametrize("shape", SHAPES, ids=str)
@pytest.mark.parametrize("dt", ["u8", "i32", "f32"])
def test_quadrants_small(fht, O, shape, dt):
    from synth import random_image
    img = random_image(shape, dt, seed=shape[0] * 1000 + shape[1])
    t = dev(img)
    for q in range(4):
        h = fht.quadrant(t, q)
        torch.cuda.synchronize()
        want = O.hough_recursive(img, q)
        check(h.view[0, 0].cpu().numpy(), want, dt != "f32")
        if dt == "f32":  # internal pin: same add tree as the float32 recursion -> bit-identical
            w32 = O.hough_recursive(img, q, dtype=np.float32)
            assert np.array_equal(h.view[0, 0].cpu().numpy(), w32)


@pytest.mark.parametrize("shape", [(8, 8), (16, 16), (3, 5), (16, 4), (5, 16), (48, 40), (64, 128), (200, 129)], ids=str)
@pytest.mark.parametrize("dt", ["u8", "f32"])
def test_full_layouts_and_shift(fht, O, shape, dt):
    from synth import random_image
    img = random_image(shape, dt, seed=sum(shape))
    t = dev(img)
    Hp, Wp = O.full_padding(*shape)
    quads = O.full_quadrants(img)
    hq = fht.full(t, "quads")
    hc = fht.full(t, "concat")
    sq = fht.fhtshift(hq)
    sc = fht.fhtshift(hc)
    fq = fht.full(t, "quads", shifted=True)
    fc = fht.full(t, "concat", shifted=True)
    torch.cuda.synchronize()
    gq = hq.view[0].cpu().numpy()
    for q in range(4):
        n = quads[q].shape[0]
        check(gq[q, :n], quads[q], dt != "f32")
        want_s = O.fhtshift_quadrant(gq[q, :n], O.QUADRANT_FRAME[q][1])
        assert np.array_equal(sq.view[0, q, :n].cpu().numpy(), want_s)
        assert np.array_equal(fq.view[0, q, :n].cpu().numpy(), want_s)
    gc = hc.view[0, 0].cpu().numpy()
    check(gc, O.full_concat(quads, Hp, Wp), dt != "f32")
    want_cs = O.fhtshift_concat(gc, Hp, Wp)
    assert np.array_equal(sc.view[0, 0].cpu().numpy(), want_cs)
    assert np.array_equal(fc.view[0, 0].cpu().numpy(), want_cs)


RANGES = [(-15, 15), (5, 40), (-30, -2), (0, 45), (-45, 0), (-80, 80), (1, 2)]


@pytest.mark.parametrize("shape", [(16, 16), (33, 17), (64, 48), (128, 128)], ids=str)
@pytest.mark.parametrize("dt", ["u8", "f32"])
def test_angle_range_small(fht, O, shape, dt):
    from synth import random_image
    img = random_image(shape, dt, seed=shape[0] + 3 * shape[1])
    t = dev(img)
    for tmin, tmax in RANGES:
        p = fht.angle_plan(*shape, tmin, tmax)
        op = O.angle_plan(*shape, tmin, tmax, k_lo=p.k_lo, k_hi=p.k_hi)   # R16: same scalars
        assert (op.W, op.w_content) == (p.W, p.w_content)
        r = fht.angle_range(t, p)
        rs = fht.fhtshift(r)
        fr = fht.angle_range(t, p, shifted=True)
        torch.cuda.synchronize()
        got = r.view[0, 0].cpu().numpy()
        check(got, O.angle_range(img, op), dt != "f32")
        want_s = O.fhtshift_range(got, op)
        assert np.array_equal(rs.view[0, 0].cpu().numpy(), want_s)
        assert np.array_equal(fr.view[0, 0].cpu().numpy(), want_s)


PRUNED_RANGES = [(-15, 15), (5, 40), (-30, -2), (0, 45), (-26, 18), (1, 2), (0, 10)]


@pytest.mark.parametrize("shape", [(16, 16), (33, 17), (64, 48), (128, 128), (200, 136)], ids=str)
@pytest.mark.parametrize("dt", ["u8", "f32"])
def test_angle_range_pruned_small(fht, O, shape, dt):
    """f2: shear-only plan, rows s <= S_max only; all cells against the oracle (same transform, first
    rows), its fhtshift standalone and fused."""
    from synth import random_image
    img = random_image(shape, dt, seed=shape[0] + 5 * shape[1])
    t = dev(img)
    for tmin, tmax in PRUNED_RANGES:
        p = fht.angle_plan(*shape, tmin, tmax, pruned=True)
        op = O.angle_plan_pruned(*shape, tmin, tmax, k_lo=p.k_lo, k_hi=p.k_hi)
        assert (op.W, op.rows) == (p.W, p.rows)
        r = fht.angle_range(t, p)
        rs = fht.fhtshift(r)
        fr, fs = fht.angle_range(t, p, pair=True)
        torch.cuda.synchronize()
        got = r.view[0, 0].cpu().numpy()
        assert got.shape == (op.rows, op.W)
        check(got, O.angle_range(img, op), dt != "f32")
        want_s = O.fhtshift_range(got, op)
        assert np.array_equal(rs.view[0, 0].cpu().numpy(), want_s)
        assert np.array_equal(fr.view[0, 0].cpu().numpy(), got)
        assert np.array_equal(fs.view[0, 0].cpu().numpy(), want_s)


HORIZONTAL_RANGES = [(-15, 15), (5, 40), (-30, -2), (0, 45), (-80, 80)]


@pytest.mark.parametrize("shape", [(16, 16), (33, 17), (64, 48), (96, 200)], ids=str)
@pytest.mark.parametrize("dt", ["u8", "f32"])
def test_angle_range_horizontal_small(fht, O, shape, dt):
    """f4: mostly-horizontal plans (the transposed image's frame, the loader gathering I[colmap][y]),
    scaled and pruned; all cells against the oracle, fhtshift fused and standalone."""
    from synth import random_image
    img = random_image(shape, dt, seed=shape[0] * 5 + shape[1])
    t = dev(img)
    for tmin, tmax in HORIZONTAL_RANGES:
        for pruned in (False, True):
            if pruned and math.tan(math.radians(tmax)) - math.tan(math.radians(tmin)) > 1.0:
                continue
            p = fht.angle_plan(*shape, tmin, tmax, pruned=pruned, horizontal=True)
            op = O.angle_plan_horizontal(*shape, tmin, tmax, pruned=pruned, k_lo=p.k_lo, k_hi=p.k_hi)
            assert (op.W, O.plan_rows(op)) == (p.W, p.rows)
            r, rs = fht.angle_range(t, p, pair=True)
            s2 = fht.fhtshift(r)
            torch.cuda.synchronize()
            got = r.view[0, 0].cpu().numpy()
            check(got, O.angle_range(img, op), dt != "f32")
            want_s = O.fhtshift_range(got, op)
            assert np.array_equal(rs.view[0, 0].cpu().numpy(), want_s)
            assert np.array_equal(s2.view[0, 0].cpu().numpy(), want_s)


def test_angle_range_horizontal_large(fht, O):
    """A 1024 x 2048 f32 image, lines within 20 deg of the horizontal: sampled cells by the direct
    pattern sums of the transposed frame, row conservation on every row."""
    from synth import random_image
    img = random_image((1024, 2048), "f32", seed=2048)
    p = fht.angle_plan(1024, 2048, -20.0, 20.0, horizontal=True)
    op = O.angle_plan_horizontal(1024, 2048, -20.0, 20.0, k_lo=p.k_lo, k_hi=p.k_hi)
    r = fht.angle_range(dev(img), p)
    torch.cuda.synchronize()
    got = r.view[0, 0].cpu().numpy()
    assert got.shape == (op.Hp, op.W)
    rng = np.random.default_rng(20)
    cells = _sample_cells(op.Hp, op.W, 1024, rng)
    check(np.array([got[a, b] for a, b in cells], dtype=np.float32), O.range_cells_direct(img, op, cells), False)
    T_total = float(O.transformed_image(img.T, op).astype(np.float64).sum())
    assert np.all(np.abs(got.astype(np.float64).sum(axis=1) - T_total) <= 1e-4 * abs(T_total) + 1e-2)


def test_angle_range_pruned_c4_image(fht, O):
    """f2 on config 4's 4096^2 f32 image, [-15, 15]: 2196 of 4096 rows; sampled cells by the direct
    pattern sums, row conservation on every row, fhtshift rows."""
    import synth
    img = synth.batch(4)[0]
    p = fht.angle_plan(4096, 4096, -15.0, 15.0, pruned=True)
    op = O.angle_plan_pruned(4096, 4096, -15.0, 15.0, k_lo=p.k_lo, k_hi=p.k_hi)
    assert (p.rows, p.W) == (op.rows, op.W) == (2196, 8192)
    r, rs = fht.angle_range(dev(img), p, pair=True)
    torch.cuda.synchronize()
    got = r.view[0, 0].cpu().numpy()
    rng = np.random.default_rng(44)
    start, length = O.range_support(op)
    extra = [(sr, int((start[sr] + dx) % op.W)) for sr in (0, 1, 1097, 2195) for dx in (-1, 0, 1, int(length[sr]) - 1)]
    cells = _sample_cells(op.rows, op.W, 2048, rng, extra)
    check(np.array([got[a, b] for a, b in cells], dtype=np.float32), O.range_cells_direct(img, op, cells), False)
    total = float(img.astype(np.float64).sum())
    assert np.all(np.abs(got.astype(np.float64).sum(axis=1) - total) <= 1e-4 * total)
    gs = rs.view[0, 0].cpu().numpy()
    k = O.fhtshift_amounts_range(op)
    for row in (0, 17, 1098, 2195):
        assert np.array_equal(gs[row], np.roll(got[row], int(k[row])))


@pytest.mark.parametrize("shape", [(33, 17), (100, 60), (64, 48), (20, 300)], ids=str)
@pytest.mark.parametrize("dt", ["u8", "f32"])
def test_quadrant_pads(fht, O, shape, dt):
    """Pads other than Hp ("extending ... by h"; R22): from 0 (lines fold: default transform +
    fold kernel) through h_frame - 1, h_frame (the paper's) to Hp + 9 (direct); every quadrant, Hough and
    fused fhtshift against the oracle's cyclic frame of that width."""
    from synth import random_image
    img = random_image(shape, dt, seed=shape[0] + 13 * shape[1])
    t = dev(img)
    for q in range(4):
        hf = shape[1] if q >= 2 else shape[0]
        Hp = O.next_pow2(hf)
        for pad in sorted({0, 1, 3, hf // 2, hf - 2, hf - 1, hf, Hp + 9} - {-1}):
            h, s = fht.quadrant(t, q, pad=pad, pair=True)
            torch.cuda.synchronize()
            got = h.view[0, 0].cpu().numpy()
            want = O.hough_recursive(img, q, pad)
            assert got.shape == want.shape
            check(got, want, dt != "f32")
            assert np.array_equal(s.view[0, 0].cpu().numpy(), O.fhtshift_quadrant(got, O.QUADRANT_FRAME[q][1], pad))
            s2 = fht.fhtshift(h)                                       # standalone kernel, same R11 rule
            torch.cuda.synchronize()
            assert np.array_equal(s2.view[0, 0].cpu().numpy(), s.view[0, 0].cpu().numpy())


def test_strided_batch_input(fht, O):
    """Non-contiguous rows (a column slice of a wider tensor) and a batch of 3."""
    from synth import random_image
    big = np.stack([random_image((40, 60), "f32", seed=s) for s in range(3)])
    t = dev(big)[:, :, 5:45]
    assert t.stride(1) == 60
    h = fht.full(t)
    torch.cuda.synchronize()
    for b in range(3):
        quads = O.full_quadrants(big[b, :, 5:45])
        for q in range(4):
            check(h.view[b, q, : quads[q].shape[0]].cpu().numpy(), quads[q], False)


def test_deterministic(fht):
    from synth import random_image
    t = dev(random_image((300, 257), "f32", seed=1))
    a = fht.full(t).view.cpu()
    b = fht.full(t).view.cpu()
    assert torch.equal(a, b)


# ------------------------------------------------------------------ the five BASELINE configs
def _sample_cells(Hp, W, n, rng, extra=()):
    s = np.concatenate([rng.integers(0, Hp, n), [0, Hp - 1, 0, Hp - 1]])
    x = np.concatenate([rng.integers(0, W, n), [0, 0, W - 1, W - 1]])
    cells = list(zip(s.tolist(), x.tolist())) + list(extra)
    return cells


def test_config1_quadrant_u8(fht, O):
    import synth
    img = synth.batch(1)[0]
    h = fht.quadrant(dev(img), fht.QA)
    torch.cuda.synchronize()
    got = h.view[0, 0].cpu().numpy()
    assert got.shape == (256, 512)
    check(got, O.hough_direct(img, O.QA), True)           # tier 1, every cell
    check(got, O.hough_recursive(img, O.QA), True)


def test_config2_full_f32_shift(fht, O):
    import synth
    img = synth.batch(2)[0]
    t = dev(img)
    h = fht.full(t)
    s = fht.fhtshift(h)
    torch.cuda.synchronize()
    got = h.view[0].cpu().numpy()
    quads = O.full_quadrants(img)
    for q in range(4):
        check(got[q], quads[q], False)
        assert np.array_equal(s.view[0, q].cpu().numpy(), O.fhtshift_quadrant(got[q], O.QUADRANT_FRAME[q][1]))


def test_config3_batch_u8(fht, O):
    import synth
    imgs = synth.batch(3)
    h = fht.full(dev(imgs))
    torch.cuda.synchronize()
    got = h.view.cpu().numpy()
    rng = np.random.default_rng(3)
    for b in range(imgs.shape[0]):
        if b in (0, 31, 63):
            quads = O.full_quadrants(imgs[b])
            for q in range(4):
                check(got[b, q], quads[q], True)
        else:
            for q in range(4):
                fr = O.quadrant_frame(imgs[b], q, square_to=(512, 512))
                cells = _sample_cells(fr.Hp, fr.W, 64, rng)
                want = O.hough_cells_direct(fr, cells)
                assert np.array_equal(np.array([got[b, q, s, x] for s, x in cells], dtype=np.int64), want)
            # row conservation on every row of every quadrant
            assert (got[b].astype(np.int64).sum(axis=2) == int(imgs[b].sum())).all()


def test_config4_range_f32(fht, O):
    import synth
    img = synth.batch(4)[0]
    p = fht.angle_plan(4096, 4096, -15.0, 15.0)
    op = O.angle_plan(4096, 4096, -15.0, 15.0, k_lo=p.k_lo, k_hi=p.k_hi)
    assert (p.W, p.w_content) == (11740, 7644)
    r = fht.angle_range(dev(img), p)
    s = fht.fhtshift(r)
    torch.cuda.synchronize()
    got = r.view[0, 0].cpu().numpy()
    rng = np.random.default_rng(4)
    start, length = O.range_support(op)
    extra = [(sr, int((start[sr] + dx) % op.W)) for sr in (0, 1, 2047, 4095) for dx in (-1, 0, 1, int(length[sr]) - 1)]
    cells = _sample_cells(op.Hp, op.W, 2048, rng, extra)
    want = O.range_cells_direct(img, op, cells)
    check(np.array([got[a, b] for a, b in cells], dtype=np.float32), want, False)
    # full rows for a few shifts, all columns
    T_total = float(np.sum(img.astype(np.float64)[np.arange(4096)[:, None],
                                                 O.scale_colmap(op.alpha, 4096, op.w_content)[None, :]]))
    sums = got.astype(np.float64).sum(axis=1)
    assert np.all(np.abs(sums - T_total) <= 1e-4 * T_total)          # row conservation
    gs = s.view[0, 0].cpu().numpy()
    k = O.fhtshift_amounts_range(op)
    for row in (0, 17, 2048, 4095):
        assert np.array_equal(gs[row], np.roll(got[row], int(k[row])))


def test_config5_batch_f32(fht, O):
    import synth
    imgs = synth.batch(5)
    h = fht.full(dev(imgs))
    s = fht.fhtshift(h)
    torch.cuda.synchronize()
    got = h.view.cpu().numpy()
    rng = np.random.default_rng(5)
    quads = O.full_quadrants(imgs[0])
    for q in range(4):
        check(got[0, q], quads[q], False)
    for b in range(1, imgs.shape[0]):
        for q in range(4):
            fr = O.quadrant_frame(imgs[b], q, square_to=(2048, 2048))
            cells = _sample_cells(fr.Hp, fr.W, 48, rng)
            want = O.hough_cells_direct(fr, cells)
            check(np.array([got[b, q, a, c] for a, c in cells], dtype=np.float32), want, False)
    gs = s.view.cpu().numpy()
    for b in (0, 15):
        for q in range(4):
            k = O.fhtshift_amounts_quadrant(2048, 4096, O.QUADRANT_FRAME[q][1])
            for row in (0, 1, 1000, 2047):
                assert np.array_equal(gs[b, q, row], np.roll(got[b, q, row], int(k[row])))


# ------------------------------------------------------------------ v2 tiling coverage
# Shapes chosen so the v2 kernels see: every pass split r = 1..6 (K = 2..12), tiles narrower
# than the 216-column maximum, several tiles with a ragged (clamped, overlapping) last tile,
# the sigma=+1 wrap at x = 0, transposed loads, and non-square frames.
V2_SHAPES = [(3, 500), (4, 300), (8, 61), (20, 1000), (70, 333), (300, 129), (513, 40), (1000, 37),
             (129, 1500), (2049, 9)]


@pytest.mark.parametrize("shape", V2_SHAPES, ids=str)
@pytest.mark.parametrize("dt", ["u8", "f32"])
def test_v2_quadrant_tiling(fht, O, shape, dt):
    from synth import random_image
    img = random_image(shape, dt, seed=7 * shape[0] + shape[1])
    t = dev(img)
    for q in range(4):
        h, s = fht.quadrant(t, q, pair=True)
        torch.cuda.synchronize()
        got = h.view[0, 0].cpu().numpy()
        want = O.hough_recursive(img, q)
        check(got, want, dt != "f32")
        sigma = O.QUADRANT_FRAME[q][1]
        assert np.array_equal(s.view[0, 0].cpu().numpy(), O.fhtshift_quadrant(got, sigma))


@pytest.mark.parametrize("shape", [(300, 700), (257, 255), (1024, 64)], ids=str)
@pytest.mark.parametrize("dt", ["u8", "i32", "f32"])
def test_v2_full_pair(fht, O, shape, dt):
    """Full transform written as (H, fhtshift(H)) by one pass, QUADS and CONCAT layouts."""
    from synth import random_image
    img = random_image(shape, dt, seed=shape[0] + 11 * shape[1])
    t = dev(img)
    Hp, Wp = O.full_padding(*shape)
    quads = O.full_quadrants(img)
    hq, sq = fht.full(t, "quads", pair=True)
    hc, sc = fht.full(t, "concat", pair=True)
    torch.cuda.synchronize()
    gq = hq.view[0].cpu().numpy()
    for q in range(4):
        n = quads[q].shape[0]
        check(gq[q, :n], quads[q], dt != "f32")
        assert np.array_equal(sq.view[0, q, :n].cpu().numpy(), O.fhtshift_quadrant(gq[q, :n], O.QUADRANT_FRAME[q][1]))
    gc = hc.view[0, 0].cpu().numpy()
    check(gc, O.full_concat(quads, Hp, Wp), dt != "f32")
    assert np.array_equal(sc.view[0, 0].cpu().numpy(), O.fhtshift_concat(gc, Hp, Wp))


@pytest.mark.parametrize("side,dt", [(2048, "u8"), (4096, "f32")], ids=["2048-u8", "4096-f32"])
def test_full_large(fht, O, side, dt):
    """Largest tilings at full size: u8 2048^2 (R = 6 pass 1 with the uint16 scratch) and f32 4096^2
    (R = 6 in both passes). Sampled cells of every quadrant by the direct pattern sums, and every row
    of every quadrant conserves the image total."""
    from synth import random_image
    img = random_image((side, side), dt, seed=side + 17)
    h = fht.full(dev(img))
    torch.cuda.synchronize()
    got = h.view[0].cpu().numpy()
    total = img.astype(np.float64).sum()
    rng = np.random.default_rng(side)
    for q in range(4):
        fr = O.quadrant_frame(img, q, square_to=(side, side))
        cells = _sample_cells(fr.Hp, fr.W, 96, rng)
        want = O.hough_cells_direct(fr, cells)
        vals = np.array([got[q, a, c] for a, c in cells], dtype=got.dtype)
        check(vals, want, dt != "f32")
        sums = got[q].astype(np.float64).sum(axis=1)
        if dt == "f32":
            assert np.all(np.abs(sums - total) <= 1e-4 * total)
        else:
            assert np.all(sums == total)


def test_v2_batch_chunks(fht, O, monkeypatch):
    """A batch split into several pass-1 scratch chunks (budget lowered to 48 MiB for the test)."""
    monkeypatch.setenv("FHT_SCRATCH_BUDGET_MB", "48")
    from synth import random_image
    imgs = np.stack([random_image((1024, 1024), "f32", seed=100 + b) for b in range(7)])
    h = fht.full(dev(imgs))
    torch.cuda.synchronize()
    assert h.launches > 4
    got = h.view.cpu().numpy()
    for b in (0, 4, 6):
        quads = O.full_quadrants(imgs[b])
        for q in range(4):
            check(got[b, q], quads[q], False)


def test_v2_aux_stream_overlap(fht, O, monkeypatch):
    """Pass 1 of chunk k+1 on an auxiliary stream overlapping pass 2 of chunk k (two scratch
    buffers): bit-identical to the single-stream schedule, and the call is complete on the
    caller's stream (budget lowered to 48 MiB so the batches need several chunks)."""
    monkeypatch.setenv("FHT_SCRATCH_BUDGET_MB", "48")
    from synth import random_image
    imgs = np.stack([random_image((1024, 1024), "f32", seed=300 + b) for b in range(7)])
    t = dev(imgs)
    h1, s1 = fht.full(t, pair=True)
    aux = torch.cuda.Stream()
    h2, s2 = fht.full(t, pair=True, aux_stream=aux)
    torch.cuda.current_stream().synchronize()          # only the caller's stream
    assert torch.equal(h1.storage, h2.storage) and torch.equal(s1.storage, s2.storage)
    quads = O.full_quadrants(imgs[5])
    for q in range(4):
        check(h2.view[5, q].cpu().numpy(), quads[q], False)
    u8 = np.stack([random_image((512, 512), "u8", seed=400 + b) for b in range(40)])
    tu = dev(u8)
    a = fht.full(tu)
    b = fht.full(tu, aux_stream=aux)
    torch.cuda.current_stream().synchronize()
    assert b.launches > 2 and torch.equal(a.storage, b.storage)


# ------------------------------------------------------------------ peaks + recovery (f3)
def _check_peaks(fht, O, H, k):
    """GPU top-k vs the oracle's rule on the SAME (GPU-computed) Hough values, every plane."""
    vals, rows, cols = fht.peaks(H, k)
    torch.cuda.synchronize()
    planes = H.view.cpu().numpy()
    v, r, c = vals.cpu().numpy(), rows.cpu().numpy(), cols.cpu().numpy()
    for b in range(planes.shape[0]):
        for q in range(planes.shape[1]):
            want = O.hough_peaks(planes[b, q], k)
            n = len(want)
            assert [(int(r[b, q, i]), int(c[b, q, i])) for i in range(n)] == [(wr, wc) for _, wr, wc in want]
            assert np.array_equal(v[b, q, :n], np.array([wv for wv, _, _ in want], dtype=v.dtype))
            assert (r[b, q, n:] == -1).all() and (c[b, q, n:] == -1).all()


@pytest.mark.parametrize("shape", [(16, 16), (33, 17), (64, 48), (128, 96)], ids=str)
@pytest.mark.parametrize("dt", ["u8", "f32"])
def test_peaks_small(fht, O, shape, dt):
    from synth import random_image
    img = random_image(shape, dt, seed=shape[0] * 3 + shape[1])
    t = dev(img)
    for k in (1, 7, 32):
        _check_peaks(fht, O, fht.full(t), k)
        _check_peaks(fht, O, fht.quadrant(t, 2), k)
    _check_peaks(fht, O, fht.full(t, layout="concat"), 16)
    _check_peaks(fht, O, fht.angle_range(t, fht.angle_plan(*shape, -15, 15)), 16)


def test_peaks_c3_batch_and_segments(fht, O):
    """Config 3 (64 u8 edge maps, planted near-horizontal lines): all 256 planes' top-16 against the
    oracle rule (sampled planes), and the recovered pattern of each image's strongest peak carries
    exactly its value (round trip on the real data: the cell sums those pixels, here 0/1 ones)."""
    import synth
    imgs = synth.batch(3)
    h = fht.full(dev(imgs))
    vals, rows, cols = fht.peaks(h, 16)
    torch.cuda.synchronize()
    planes = h.view.cpu().numpy()
    v, r, c = vals.cpu().numpy(), rows.cpu().numpy(), cols.cpu().numpy()
    rng = np.random.default_rng(33)
    for b in rng.choice(64, 6, replace=False):
        for q in range(4):
            want = O.hough_peaks(planes[b, q], 16)
            assert [(int(r[b, q, i]), int(c[b, q, i]), int(v[b, q, i])) for i in range(16)] == \
                   [(wr, wc, int(wv)) for wv, wr, wc in want]
    for b in range(0, 64, 9):
        q = int(np.argmax(v[b, :, 0]))
        seg = fht.cell_segment(h, int(r[b, q, 0]), int(c[b, q, 0]), slot=q)
        _, _, pix = O.cell_segment("full", 512, 512, int(r[b, q, 0]), int(c[b, q, 0]), quadrant=q)
        assert seg["npix"] == len(pix) and (seg["first"], seg["last"]) == (pix[0], pix[-1])
        assert int(sum(int(imgs[b][y, x]) for x, y in pix)) == int(v[b, q, 0])


def test_graph_replay_equals_eager(fht, O):
    """A captured step (pass pair with PDL, fused fhtshift, the two-stream orientation split) replays
    to the same bits as the eager call; new input values flow through the same graph."""
    import synth
    img = synth.batch(2)[0]
    t = dev(img)
    h0, s0 = fht.full(t, pair=True)
    h, s = fht.full(t, pair=True)
    ws = torch.empty(fht.workspace_bytes(fht.FHT_MODE_FULL, fht._image(t)[0], None), dtype=torch.uint8, device="cuda")
    aux = torch.cuda.Stream()
    g = fht.Graph(lambda: fht.full(t, pair=True, out=h, out_shifted=s, workspace=ws, aux_stream=aux))
    h.storage.zero_()
    s.storage.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(h.storage, h0.storage) and torch.equal(s.storage, s0.storage)
    t.copy_(t.flip(0))                      # new values, same buffer
    g.replay()
    h1, s1 = fht.full(t, pair=True)
    torch.cuda.synchronize()
    assert torch.equal(h.storage, h1.storage) and torch.equal(s.storage, s1.storage)


# ------------------------------------------------------------------ round 2: the benched calls themselves
# bench.py times these exact calls (same arguments, streams and graph capture); here they are compared
# with the oracle on EVERY cell of every output. Oracle work runs in a fork pool of host processes
# (numpy only; the children never touch CUDA).
_G = {}


def _pool_map(fn, items):
    import multiprocessing as mp
    import os
    n = max(1, min(len(items), 16, len(os.sched_getaffinity(0))))
    with mp.get_context("fork").Pool(n) as pool:
        errs = [r for r in pool.imap_unordered(fn, items) if r is not None]
    assert not errs, errs[:5]


def _tol_err(got, want):
    err = np.abs(got.astype(np.float64) - want)
    bad = err > ATOL + RTOL * np.abs(want)
    return None if not bad.any() else f"{int(bad.sum())} cells out of tolerance, max err {err.max()}"


def _full_unit(args):
    """(b, q): oracle quadrant q of image b vs the GPU planes in _G; plain and fhtshift-ed outputs."""
    from oracle import fht_oracle as O
    b, q = args
    img = _G["imgs"][b]
    Hp, Wp = O.full_padding(*img.shape)
    fr = O.quadrant_frame(img, q, square_to=(Hp, Wp))
    want = O.hough_of_frame_recursive(fr)
    n = want.shape[0]
    integer = _G["integer"]
    msgs = []
    if "h" in _G:
        got = _G["h"][b, q, :n]
        if integer:
            if not np.array_equal(got.astype(np.int64), want):
                msgs.append(f"img {b} q {q}: plain mismatch")
        else:
            e = _tol_err(got, want)
            if e:
                msgs.append(f"img {b} q {q}: plain {e}")
    if "s" in _G:
        gs = _G["s"][b, q, :n]
        want_s = O.fhtshift_quadrant(want, fr.sigma)
        e = (None if np.array_equal(gs.astype(np.int64), want_s) else "mismatch") if integer else _tol_err(gs, want_s)
        if e:
            msgs.append(f"img {b} q {q}: shifted {e}")
        if "h" in _G and not np.array_equal(gs, O.fhtshift_quadrant(_G["h"][b, q, :n], fr.sigma)):
            msgs.append(f"img {b} q {q}: shifted is not the exact rotation of the plain output")
    return "; ".join(msgs) or None


def test_config1_bench_step(fht, O):
    """C1 as bench.py times it: the QA call captured in a CUDA graph and replayed."""
    import synth
    img = synth.batch(1)[0]
    t = dev(img)
    h = fht.quadrant(t, fht.QA)
    ws = torch.empty(fht.workspace_bytes(fht.FHT_MODE_QUADRANT, fht._image(t)[0]), dtype=torch.uint8, device="cuda")
    g = fht.Graph(lambda: fht.quadrant(t, fht.QA, out=h, workspace=ws))
    h.storage.zero_()
    g.replay()
    torch.cuda.synchronize()
    check(h.view[0, 0].cpu().numpy(), O.hough_direct(img, O.QA), True)


def test_config2_bench_step(fht, O):
    """C2 as bench.py times it: full(pair=True, aux_stream) -- the two-stream orientation split --
    captured in a CUDA graph; both outputs, every cell, against the oracle."""
    import synth
    img = synth.batch(2)[0]
    t = dev(img)
    h, s = fht.full(t, pair=True)
    ws = torch.empty(fht.workspace_bytes(fht.FHT_MODE_FULL, fht._image(t)[0]), dtype=torch.uint8, device="cuda")
    aux = torch.cuda.Stream()
    g = fht.Graph(lambda: fht.full(t, pair=True, out=h, out_shifted=s, workspace=ws, aux_stream=aux))
    h.storage.zero_()
    s.storage.zero_()
    g.replay()
    torch.cuda.synchronize()
    _G.clear()
    _G.update(imgs=img[None], integer=False, h=h.view.cpu().numpy(), s=s.view.cpu().numpy())
    _pool_map(_full_unit, [(0, q) for q in range(4)])


def test_config3_bench_step(fht, O):
    """C3 as bench.py times it: full(aux_stream) over the 64-image u8 batch; all 256 planes, every cell,
    bit-exact."""
    import synth
    imgs = synth.batch(3)
    aux = torch.cuda.Stream()
    h = fht.full(dev(imgs), aux_stream=aux)
    torch.cuda.synchronize()
    _G.clear()
    _G.update(imgs=imgs, integer=True, h=h.view.cpu().numpy())
    _pool_map(_full_unit, [(b, q) for b in range(imgs.shape[0]) for q in range(4)])


def test_config5_bench_step(fht, O):
    """C5 as bench.py times it: full(pair=True, aux_stream) over the 16 x 2048^2 batch; both outputs of
    all 16 images, every cell, against the oracle. The single-destination step (shifted=True) must
    write the same bits as the pair's fhtshift output."""
    import synth
    imgs = synth.batch(5)
    t = dev(imgs)
    aux = torch.cuda.Stream()
    h, s = fht.full(t, pair=True, aux_stream=aux)
    s1 = fht.full(t, shifted=True, aux_stream=aux)
    torch.cuda.synchronize()
    assert torch.equal(s1.storage, s.storage)
    del s1, t
    _G.clear()
    _G.update(imgs=imgs, integer=False, h=h.view.cpu().numpy(), s=s.view.cpu().numpy())
    del h, s
    torch.cuda.empty_cache()
    _pool_map(_full_unit, [(b, q) for b in range(imgs.shape[0]) for q in range(4)])
    _G.clear()


def test_config4_bench_step(fht, O):
    """C4 as bench.py times it: angle_range(t, -15, 15, pair=True) (fht_angle_range builds the §4 plan);
    both outputs, every cell, against the oracle's tier-2 recursion on the materialised T."""
    import synth
    img = synth.batch(4)[0]
    r, rs = fht.angle_range(dev(img), -15.0, 15.0, pair=True)
    torch.cuda.synchronize()
    p = r.plan
    assert (p.W, p.w_content, p.rows) == (11740, 7644, 4096)
    op = O.angle_plan(4096, 4096, -15.0, 15.0, k_lo=p.k_lo, k_hi=p.k_hi)
    want = O.angle_range(img, op)
    got = r.view[0, 0].cpu().numpy()
    check(got, want, False)
    gs = rs.view[0, 0].cpu().numpy()
    check(gs, O.fhtshift_range(want, op), False)
    assert np.array_equal(gs, O.fhtshift_range(got, op))


@pytest.mark.parametrize("dt", ["f32", "u8"])
def test_angle_range_steep_colmap_fallback(fht, O, dt):
    """A steep narrow range on a 2048-row image: [-85, -84.6] deg has g = alpha (-k_lo) ~ 13.4 columns
    per row, so a 64-row strip's transformed columns span ~860 image columns -- beyond the 512-entry
    shared-memory colmap slice, the pass-1 loader's global colmap branch. Every cell vs the oracle."""
    from synth import random_image
    img = random_image((2048, 40), dt, seed=8584)
    p = fht.angle_plan(2048, 40, -85.0, -84.6)
    assert p.alpha >= 1.0 and p.g * 63 > 512
    r, rs = fht.angle_range(dev(img), -85.0, -84.6, pair=True)
    torch.cuda.synchronize()
    op = O.angle_plan(2048, 40, -85.0, -84.6, k_lo=p.k_lo, k_hi=p.k_hi)
    assert (op.W, op.w_content) == (p.W, p.w_content)
    want = O.angle_range(img, op)
    got = r.view[0, 0].cpu().numpy()
    check(got, want, dt != "f32")
    assert np.array_equal(rs.view[0, 0].cpu().numpy(), O.fhtshift_range(got, op))


@pytest.mark.parametrize("shape", [(3, 5), (64, 64), (100, 37), (300, 700), (257, 255), (1024, 64)], ids=str)
def test_i32_signed_large_values(fht, O, shape):
    """int32 input with negative and large values (|v| <= (2^31 - 1) / P, so every sum fits int32):
    quadrants and the full transform, bit-exact against the int64 oracle."""
    from synth import random_image
    P = max(O.full_padding(*shape))
    img = random_image(shape, "i32w", seed=shape[0] * 3 + shape[1], bound=(2 ** 31 - 1) // P)
    assert img.min() < -(2 ** 20) // P and img.max() > (2 ** 20) // P
    t = dev(img)
    for q in range(4):
        h, s = fht.quadrant(t, q, pair=True)
        torch.cuda.synchronize()
        want = O.hough_recursive(img, q)
        got = h.view[0, 0].cpu().numpy()
        check(got, want, True)
        assert np.array_equal(s.view[0, 0].cpu().numpy(), O.fhtshift_quadrant(got, O.QUADRANT_FRAME[q][1]))
    hq, sq = fht.full(t, pair=True)
    torch.cuda.synchronize()
    quads = O.full_quadrants(img)
    for q in range(4):
        n = quads[q].shape[0]
        check(hq.view[0, q, :n].cpu().numpy(), quads[q], True)
        check(sq.view[0, q, :n].cpu().numpy(), O.fhtshift_quadrant(quads[q], O.QUADRANT_FRAME[q][1]), True)


# ------------------------------------------------------------------ the pipelined kernel (fht_pipe.cuh)
PIPE_VARIANTS = [{}, {"FHT_PIPE_D": "1", "FHT_PIPE_NBUF": "2"}, {"FHT_PIPE_D": "3", "FHT_PIPE_NBUF": "4"},
                 {"FHT_PIPE_UNIT_MB": "1"}]


@pytest.mark.parametrize("shape,dt,batch", [((256, 256), "u8", 3), ((300, 500), "f32", 1), ((512, 512), "u8", 6),
                                            ((1024, 1024), "f32", 2), ((2048, 2048), "f32", 1), ((4096, 4096), "f32", 1),
                                            ((700, 900), "i32", 2)], ids=str)
def test_pipe_matches_two_launch_and_oracle(fht, O, monkeypatch, shape, dt, batch):
    """One persistent launch for both passes (pass 1 of unit u + D beside pass 2 of unit u, a ring of NBUF
    scratch buffers): bit-identical to the two-launch schedule for every lookahead / ring / unit size
    (including the tight ring D = 1, NBUF = 2 whose pass-1 items wait on buffer reuse), one launch per
    call, and every cell of image 0 against the oracle."""
    from synth import random_image
    imgs = np.stack([random_image(shape, dt, seed=shape[0] + b) for b in range(batch)])
    t = dev(imgs)
    monkeypatch.setenv("FHT_PIPE", "0")
    h0, s0 = fht.full(t, pair=True)
    torch.cuda.synchronize()
    assert h0.launches >= 2
    for env in PIPE_VARIANTS:
        monkeypatch.setenv("FHT_PIPE", "1")
        for k in ("FHT_PIPE_D", "FHT_PIPE_NBUF", "FHT_PIPE_UNIT_MB"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        h, s = fht.full(t, pair=True)
        q1 = fht.quadrant(t, fht.QC)
        torch.cuda.synchronize()
        assert h.launches == 1, env
        assert torch.equal(h.storage, h0.storage) and torch.equal(s.storage, s0.storage), env
    quads = O.full_quadrants(imgs[0])
    got = h.view[0].cpu().numpy()
    for q in range(4):
        n = quads[q].shape[0]
        check(got[q, :n], quads[q], dt != "f32")
    if batch > 1:   # one quadrant of a batch: units = images
        check(q1.view[batch - 1, 0].cpu().numpy(), O.hough_recursive(imgs[batch - 1], O.QC), dt != "f32")


# ------------------------------------------------------------------ staggered pass pairs (fht_dual.cuh)
@pytest.mark.parametrize("shape,dt,batch,imgs", [((512, 512), "u8", 5, "1"), ((512, 512), "u8", 7, "2"),
                                                 ((1024, 1024), "f32", 3, "1"), ((2048, 2048), "f32", 3, "1"),
                                                 ((2048, 2048), "f32", 5, "2"), ((4096, 4096), "f32", 2, "1"),
                                                 ((700, 900), "i32", 3, "1"), ((1000, 1024), "f32", 4, "3")], ids=str)
def test_dual_matches_two_launch_and_oracle(fht, O, monkeypatch, shape, dt, batch, imgs):
    """Pass 1 of chunk k beside pass 2 of chunk k - 1 in one grid (FHT_DUAL_IMGS images per chunk, two
    scratch buffers, a ragged last chunk when the batch does not divide): bit-identical to the two-launch
    schedule, nchunks + 1 launches, both outputs, every cell of the last image against the oracle."""
    from synth import random_image
    ims = np.stack([random_image(shape, dt, seed=shape[1] + 7 * b) for b in range(batch)])
    t = dev(ims)
    monkeypatch.delenv("FHT_DUAL_IMGS", raising=False)
    h0, s0 = fht.full(t, pair=True)
    torch.cuda.synchronize()
    monkeypatch.setenv("FHT_DUAL_IMGS", imgs)
    h, s = fht.full(t, pair=True)
    torch.cuda.synchronize()
    nch = -(-batch // int(imgs))
    assert h.launches == nch + 1
    assert torch.equal(h.storage, h0.storage) and torch.equal(s.storage, s0.storage)
    quads = O.full_quadrants(ims[batch - 1])
    got = h.view[batch - 1].cpu().numpy()
    for q in range(4):
        n = quads[q].shape[0]
        check(got[q, :n], quads[q], dt != "f32")


# ------------------------------------------------------------------ one image over several ranks
def _emulated_shards(fht, t, world, p2p):
    """All `world` ranks of a sharded transform run in this process on one GPU (their kernels do not
    wait on each other, so this is not a multi-rank emulation of waiting kernels): pass 1 of every rank,
    the all-to-all done as chunk copies (or, p2p, pass 1 storing straight into the receive buffers as
    the peer-memory path does), pass 2 of every rank. Returns the ranks' (band, band_shifted)."""
    from paper_1811_06378_b200 import sharding as SH
    shs = [SH.shard_describe(t, world, r) for r in range(world)]
    ch = shs[0].chunk_bytes
    recv = [torch.empty(shs[0].recv_bytes, dtype=torch.uint8, device=t.device) for _ in range(world)]
    if p2p:
        for g in range(world):
            SH.shard_pass1(t, shs[g], [recv[h].data_ptr() + g * ch for h in range(world)])
    else:
        send = [torch.empty(shs[0].send_bytes, dtype=torch.uint8, device=t.device) for _ in range(world)]
        for g in range(world):
            SH.shard_pass1(t, shs[g], [send[g].data_ptr() + h * ch for h in range(world)])
        for g in range(world):
            for h in range(world):
                recv[h][g * ch:(g + 1) * ch].copy_(send[g][h * ch:(h + 1) * ch])
    return [SH.shard_pass2(t, shs[h], recv[h], pair=True) for h in range(world)]


@pytest.mark.parametrize("shape,dt,batch,world", [((1024, 1024), "f32", 1, 2), ((1024, 1024), "f32", 1, 8),
                                                  ((512, 512), "u8", 3, 4), ((2048, 2048), "f32", 1, 4),
                                                  ((300, 500), "i32", 2, 2), ((256, 256), "u8", 1, 8)], ids=str)
@pytest.mark.parametrize("p2p", [False, True], ids=["nccl-layout", "p2p-stores"])
def test_shard_bands_equal_full(fht, O, shape, dt, batch, world, p2p):
    """Concatenated bands of the sharded transform are bit-identical to the one-GPU full transform (same
    single IEEE add per output, any split of the levels), plain and fhtshift-ed; image 0 against the oracle;
    the standalone fhtshift of a band (row0) equals the fused one."""
    from synth import random_image
    imgs = np.stack([random_image(shape, dt, seed=shape[0] * 3 + b) for b in range(batch)])
    t = dev(imgs)
    h, s = fht.full(t, pair=True)
    bands = _emulated_shards(fht, t, world, p2p)
    torch.cuda.synchronize()
    rows = bands[0][0].desc.rows
    for r, (hb, sb) in enumerate(bands):
        assert hb.desc.row0 == r * rows and hb.launches == 1
        assert torch.equal(hb.view, h.view[:, :, r * rows:(r + 1) * rows])
        assert torch.equal(sb.view, s.view[:, :, r * rows:(r + 1) * rows])
    s1 = fht.fhtshift(bands[-1][0])
    torch.cuda.synchronize()
    assert torch.equal(s1.view, bands[-1][1].view)
    quads = O.full_quadrants(imgs[0])
    got = torch.cat([hb.view for hb, _ in bands], dim=2)[0].cpu().numpy()
    for q in range(4):
        n = quads[q].shape[0]
        check(got[q, :n], quads[q], dt != "f32")


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_shard_two_devices_nccl():
    """Two ranks on two GPUs over NCCL (torchrun-free: spawned processes): each rank's band equals the
    corresponding rows of the one-GPU transform. Skipped on one-GPU boxes."""
    import socket
    import torch.multiprocessing as mp
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nccl_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def _nccl_shard_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    import paper_1811_06378_b200 as F
    from synth import random_image
    t = torch.from_numpy(random_image((1024, 1024), "f32", seed=5)).cuda()
    hb, sb = F.full_sharded(t, pair=True)
    h, s = F.full(t, pair=True)
    torch.cuda.synchronize()
    rows = hb.desc.rows
    ok = torch.equal(hb.view, h.view[:, :, rank * rows:(rank + 1) * rows]) and \
        torch.equal(sb.view, s.view[:, :, rank * rows:(rank + 1) * rows])
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


def _same_planes(x, y, shape):
    """Bitwise equality of two QUADS views [B][4][rows][W] on the rows each quadrant holds (QA/QB: Hp, QC/QD: Wp; for
    non-square frames the planes' remaining rows are never written)."""
    from oracle import fht_oracle as _O
    Hp, Wp = _O.full_padding(*shape)
    return all(np.array_equal(x[:, q, :n].view(np.int32), y[:, q, :n].view(np.int32))
               for q, n in ((0, Hp), (1, Hp), (2, Wp), (3, Wp)))


@pytest.mark.parametrize("shape,dt,batch", [((2048, 2048), "f32", 2), ((2048, 2048), "i32", 1), ((4096, 4096), "f32", 1),
                                            ((1500, 1504), "f32", 3), ((2048, 1056), "i32", 2), ((1100, 2080), "f32", 1),
                                            ((3000, 2016), "f32", 1)],
                         ids=lambda v: str(v))
def test_persistent_pass1(fht, O, monkeypatch, shape, dt, batch):
    """The persistent pass 1 (k_p1p: 64-row strips of 4-byte images, prefetched loads, warp-owned half-slot
    stores) against k_p1 on the same call: both outputs bit-identical, over square / non-square / non-power-of-two
    frames, batches and the chunked schedule; and sampled cells of image 0 against the direct pattern sums."""
    from synth import random_image
    h_, w_ = shape
    imgs = np.stack([random_image(shape, dt, seed=6100 + 7 * b + h_) for b in range(batch)])
    if dt == "i32":  # signed, large
        imgs = (imgs.astype(np.int64) * 4001 - 500000).astype(np.int32)
    t = dev(imgs)
    monkeypatch.setenv("FHT_P1_PERSIST", "0")
    h0, s0 = fht.full(t, pair=True)
    torch.cuda.synchronize()
    a0, b0 = h0.view.cpu().numpy(), s0.view.cpu().numpy()
    del h0, s0
    monkeypatch.setenv("FHT_P1_PERSIST", "1")
    h1, s1 = fht.full(t, pair=True)
    torch.cuda.synchronize()
    a1, b1 = h1.view.cpu().numpy(), s1.view.cpu().numpy()
    assert _same_planes(a0, a1, shape)
    assert _same_planes(b0, b1, shape)
    for _ in range(3):  # repeated: a shared-memory reuse race in the tile loop showed up about once in three runs
        hr = fht.full(t, out=h1)
        torch.cuda.synchronize()
        assert _same_planes(hr.view.cpu().numpy(), a1, shape)
    if batch > 1:  # several chunks (two scratch buffers)
        monkeypatch.setenv("FHT_SCRATCH_BUDGET_MB", "80")
        h2 = fht.full(t)
        torch.cuda.synchronize()
        assert _same_planes(h2.view.cpu().numpy(), a1, shape)
        # the chunks pipelined over an auxiliary stream (pass 1 of chunk k + 1 beside pass 2 of chunk k)
        h3, s3 = fht.full(t, pair=True, aux_stream=torch.cuda.Stream())
        torch.cuda.synchronize()
        assert h3.launches >= 4
        assert _same_planes(h3.view.cpu().numpy(), a1, shape)
        assert _same_planes(s3.view.cpu().numpy(), b1, shape)
    rng = np.random.default_rng(h_ * 3 + w_)
    for q in range(4):
        fr = O.quadrant_frame(imgs[0], q, square_to=O.full_padding(h_, w_))
        cells = _sample_cells(fr.Hp, fr.W, 48, rng)
        want = O.hough_cells_direct(fr, cells)
        vals = np.array([a1[0, q, a, c] for a, c in cells], dtype=a1.dtype)
        check(vals, want, dt != "f32")


@pytest.mark.parametrize("shape,dt,rng_deg,pruned", [((4096, 4096), "f32", (-15.0, 15.0), False),
                                                     ((4096, 4096), "f32", (-15.0, 15.0), True),
                                                     ((2048, 1200), "i32", (5.0, 30.0), False),
                                                     ((1700, 2304), "f32", (-40.0, -10.0), False)], ids=lambda v: str(v))
def test_persistent_pass1_range(fht, monkeypatch, shape, dt, rng_deg, pruned):
    """The §4 range loader inside the persistent pass 1 (k_p1p, 64-row strips) against k_p1 on the same call:
    the range Hough image and its fhtshift bit-identical (the oracle comparisons of these frames are
    test_config4_* and test_range_*; this pins the two kernels to each other on more frames), repeated."""
    from synth import random_image
    img = random_image(shape, dt, seed=7300 + shape[0] + shape[1])
    t = dev(img)
    plan = fht.angle_plan(shape[0], shape[1], rng_deg[0], rng_deg[1], pruned=pruned)
    monkeypatch.setenv("FHT_P1_PERSIST", "0")
    h0, s0 = fht.angle_range(t, plan, pair=True)
    torch.cuda.synchronize()
    a0, b0 = h0.view.cpu().numpy(), s0.view.cpu().numpy()
    monkeypatch.setenv("FHT_P1_PERSIST", "1")
    for _ in range(3):
        h1, s1 = fht.angle_range(t, plan, pair=True)
        torch.cuda.synchronize()
        assert np.array_equal(h1.view.cpu().numpy().view(np.int32), a0.view(np.int32))
        assert np.array_equal(s1.view.cpu().numpy().view(np.int32), b0.view(np.int32))


@pytest.mark.parametrize("shape,batch", [((512, 512), 5), ((256, 256), 1), ((300, 384), 2), ((512, 640), 2),
                                         ((200, 128), 3)], ids=lambda v: str(v))
def test_persistent_pass1_u8(fht, O, monkeypatch, shape, batch):
    """The persistent pass 1 for 16-row strips of u8 images (k_p1p8: per-warp prefetched row boxes, transposed tiles
    read as words of the untransposed block, uint16 scratch through per-warp slots) against k_p1 on the same call:
    both outputs bit-identical, repeated; and sampled cells of image 0 against the direct pattern sums."""
    from synth import random_image
    h_, w_ = shape
    imgs = np.stack([random_image(shape, "u8", seed=8100 + 5 * b + w_) for b in range(batch)])
    t = dev(imgs)
    monkeypatch.setenv("FHT_P1_PERSIST", "0")
    h0, s0 = fht.full(t, pair=True)
    torch.cuda.synchronize()
    a0, b0 = h0.view.cpu().numpy(), s0.view.cpu().numpy()
    monkeypatch.setenv("FHT_P1_PERSIST", "1")
    for _ in range(3):
        h1, s1 = fht.full(t, pair=True)
        torch.cuda.synchronize()
        assert _same_planes(h1.view.cpu().numpy(), a0, shape)
        assert _same_planes(s1.view.cpu().numpy(), b0, shape)
    rng = np.random.default_rng(h_ + 7 * w_)
    for q in range(4):
        fr = O.quadrant_frame(imgs[0], q, square_to=O.full_padding(h_, w_))
        cells = _sample_cells(fr.Hp, fr.W, 48, rng)
        want = O.hough_cells_direct(fr, cells)
        vals = np.array([a0[0, q, a, c] for a, c in cells], dtype=a0.dtype)
        check(vals, want, True)
