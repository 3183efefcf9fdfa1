"""CPU tests of the C ABI boundary: the library loads, exports every symbol include/fht.h
declares, and the host-only calls (describe, workspace sizing, plan, argument checks) behave
as documented. No compute call runs here (no GPU)."""
import ctypes
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_1811_06378_b200 import _lib as L
    return L


def test_header_symbols_exported():
    L = _lib()
    hdr = open(os.path.join(ROOT, "include", "fht.h")).read()
    decl = set(re.findall(r"^(?:int|size_t|const char\*)\s+(\w+)\s*\(", hdr, flags=re.M))
    assert decl == set(L.EXPORTED), decl
    for name in decl:
        assert hasattr(L.lib, name)


def test_struct_sizes_match_header(tmp_path):
    """The ctypes mirrors have the C compiler's sizeof for every struct include/fht.h declares."""
    import subprocess
    L = _lib()
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "fht.h"\nint main(void) { printf("%zu %zu %zu %zu", '
                   'sizeof(fht_image), sizeof(fht_angle_plan_t), sizeof(fht_hough), sizeof(fht_exec_opts)); return 0; }\n')
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(tmp_path / "sz")], check=True)
    got = [int(x) for x in subprocess.run([str(tmp_path / "sz")], capture_output=True, text=True, check=True).stdout.split()]
    assert got == [ctypes.sizeof(L.FhtImage), ctypes.sizeof(L.FhtAnglePlan), ctypes.sizeof(L.FhtHough),
                   ctypes.sizeof(L.FhtExecOpts)]
    assert ctypes.sizeof(L.FhtAnglePlan) == 6 * 8 + 9 * 8


def _img(L, h, w, b=1, dt=2, data=4096):
    img = L.FhtImage()
    img.data, img.dtype, img.batch, img.h, img.w = data, dt, b, h, w
    img.row_stride, img.batch_stride = w, h * w
    return img


@pytest.mark.parametrize("h,w", [(1024, 1024), (512, 512), (3, 5), (100, 37)])
def test_describe_shapes(h, w):
    L = _lib()
    img = _img(L, h, w)
    Hp, Wp = 1 << (h - 1).bit_length(), 1 << (w - 1).bit_length()
    d = L.FhtHough()
    assert L.lib.fht_hough_describe(L.FHT_MODE_FULL, L.FHT_LAYOUT_QUADS, 0, ctypes.byref(img), None, ctypes.byref(d)) == 0
    assert (d.nquad, d.rows, d.cols) == (4, max(Hp, Wp), Hp + Wp)
    assert L.lib.fht_hough_describe(L.FHT_MODE_FULL, L.FHT_LAYOUT_CONCAT, 0, ctypes.byref(img), None, ctypes.byref(d)) == 0
    assert (d.nquad, d.rows, d.cols) == (1, 2 * (Hp + Wp) - 3, Hp + Wp)
    assert L.lib.fht_hough_describe(L.FHT_MODE_QUADRANT, 0, 0, ctypes.byref(img), None, ctypes.byref(d)) == 0
    assert (d.rows, d.cols) == (Hp, w + Hp)
    assert L.lib.fht_hough_describe(L.FHT_MODE_QUADRANT, 0, 2, ctypes.byref(img), None, ctypes.byref(d)) == 0
    assert (d.rows, d.cols) == (Wp, h + Wp)
    assert d.row_stride % 4 == 0 and d.row_stride >= d.cols


def test_plan_matches_oracle_rule():
    from oracle import fht_oracle as O
    L = _lib()
    for h, w, a, b in [(4096, 4096, -15, 15), (64, 48, 5, 40), (33, 17, -45, 0), (16, 16, 0, 45), (32, 32, -80, 80)]:
        p = L.FhtAnglePlan()
        assert L.lib.fht_angle_plan(h, w, a, b, ctypes.byref(p)) == 0
        o = O.angle_plan(h, w, a, b)
        assert (p.k_lo, p.k_hi, p.alpha, p.g) == (o.k_lo, o.k_hi, o.alpha, o.g)
        assert (p.Hp, p.w_content, p.W) == (o.Hp, o.w_content, o.W)
        e = O.shear_offsets(o.g, h)
        assert (p.e_min, p.e_max) == (e.min(), e.max())


def test_pruned_plan_matches_oracle_rule():
    """fht_angle_plan_make_pruned (f2): same scalars, rows and W' as the oracle's pruned plan."""
    from oracle import fht_oracle as O
    L = _lib()
    for h, w, a, b in [(4096, 4096, -15, 15), (64, 48, 5, 40), (33, 17, -20, 0), (16, 16, 0, 45), (128, 96, -26, 18)]:
        p = L.FhtAnglePlan()
        assert L.lib.fht_angle_plan_make_pruned(h, w, a, b, ctypes.byref(p)) == 0
        o = O.angle_plan_pruned(h, w, a, b)
        assert (p.k_lo, p.k_hi, p.alpha, p.g) == (o.k_lo, o.k_hi, 1.0, o.g)
        assert (p.Hp, p.w_content, p.W, p.rows) == (o.Hp, o.w_content, o.W, o.rows)
        d = L.FhtHough()
        img = _img(L, h, w)
        assert L.lib.fht_hough_describe(L.FHT_MODE_RANGE, 0, 0, ctypes.byref(img), ctypes.byref(p), ctypes.byref(d)) == 0
        assert (d.rows, d.cols) == (o.rows, o.W)
    p = L.FhtAnglePlan()
    assert L.lib.fht_angle_plan(64, 64, -15, 15, ctypes.byref(p)) == 0 and p.rows == p.Hp
    assert L.lib.fht_angle_plan_make_pruned(64, 64, -30, 30, ctypes.byref(p)) == -5   # k_hi - k_lo > 1


def test_plan_ex_matches_oracle():
    """fht_angle_plan_make_ex: HORIZONTAL builds the plan on the transposed image (frame h, w swapped),
    PRUNED as before, both combined; descriptors follow the frame."""
    from oracle import fht_oracle as O
    L = _lib()
    for h, w, a, b, flags in [(64, 48, -15, 15, 2), (33, 17, 5, 40, 2), (128, 96, -20, 10, 3), (16, 16, 0, 45, 2)]:
        p = L.FhtAnglePlan()
        assert L.lib.fht_angle_plan_make_ex(h, w, a, b, flags, ctypes.byref(p)) == 0
        o = O.angle_plan_horizontal(h, w, a, b, pruned=bool(flags & 1))
        assert p.transposed == 1 and (p.h, p.w) == (o.h, o.w) == (w, h)
        assert (p.k_lo, p.k_hi, p.alpha, p.g) == (o.k_lo, o.k_hi, o.alpha, o.g)
        assert (p.Hp, p.w_content, p.W, p.rows) == (o.Hp, o.w_content, o.W, O.plan_rows(o))
        d = L.FhtHough()
        img = _img(L, h, w)
        assert L.lib.fht_hough_describe(L.FHT_MODE_RANGE, 0, 0, ctypes.byref(img), ctypes.byref(p), ctypes.byref(d)) == 0
        assert (d.rows, d.cols) == (O.plan_rows(o), o.W)
        bad = _img(L, w, h) if w != h else None
        if bad is not None:   # the plan's frame is the transposed image: an h x w plan does not fit w x h
            assert L.lib.fht_hough_describe(L.FHT_MODE_RANGE, 0, 0, ctypes.byref(bad), ctypes.byref(p),
                                            ctypes.byref(d)) == -1
    p = L.FhtAnglePlan()
    assert L.lib.fht_angle_plan_make_ex(16, 16, -10, 10, 4, ctypes.byref(p)) == -1    # unknown flag


def test_plan_errors():
    L = _lib()
    p = L.FhtAnglePlan()
    assert L.lib.fht_angle_plan(16, 16, 10, 10, ctypes.byref(p)) == -1
    assert L.lib.fht_angle_plan(16, 16, -90, 10, ctypes.byref(p)) == -1
    assert L.lib.fht_angle_plan(16, 16, 20, 10, ctypes.byref(p)) == -1
    assert L.lib.fht_angle_plan(1, 1, -89.9, 89.9, ctypes.byref(p)) == -1      # alpha * w < 1
    assert L.lib.fht_angle_plan(0, 16, -10, 10, ctypes.byref(p)) == -1


def test_argument_errors_are_synchronous():
    """Checks that return before anything is enqueued (no GPU needed)."""
    L = _lib()
    img = _img(L, 16, 16)
    d = L.FhtHough()
    assert L.lib.fht_hough_describe(1, 0, 0, ctypes.byref(img), None, ctypes.byref(d)) == 0
    d.data = 1 << 20
    ws_n = L.lib.fht_workspace_bytes(1, ctypes.byref(img), None)
    assert ws_n > 0
    assert L.lib.fht_full(None, 0, ctypes.byref(d), None, 1 << 24, ws_n, None, None) == -1         # NULL image
    bad = _img(L, 16, 16, dt=7)
    assert L.lib.fht_full(ctypes.byref(bad), 0, ctypes.byref(d), None, 1 << 24, ws_n, None, None) == -2
    zero = _img(L, 0, 16)
    assert L.lib.fht_full(ctypes.byref(zero), 0, ctypes.byref(d), None, 1 << 24, ws_n, None, None) == -1
    d2 = L.FhtHough.from_buffer_copy(d)
    d2.rows += 1
    assert L.lib.fht_full(ctypes.byref(img), 0, ctypes.byref(d2), None, 1 << 24, ws_n, None, None) == -3
    assert L.lib.fht_full(ctypes.byref(img), 1, ctypes.byref(d), None, 1 << 24, ws_n, None, None) == -3   # layout mismatch
    assert L.lib.fht_full(ctypes.byref(img), 0, ctypes.byref(d), None, None, ws_n, None, None) == -6
    assert L.lib.fht_full(ctypes.byref(img), 0, ctypes.byref(d), None, 1 << 24, 16, None, None) == -6
    alias = _img(L, 16, 16, data=d.data)
    assert L.lib.fht_full(ctypes.byref(alias), 0, ctypes.byref(d), None, 1 << 24, ws_n, None, None) == -1
    odd = _img(L, 16, 16, data=4098)
    assert L.lib.fht_full(ctypes.byref(odd), 0, ctypes.byref(d), None, 1 << 24, ws_n, None, None) == -4
    dq = L.FhtHough()
    assert L.lib.fht_hough_describe(0, 0, 0, ctypes.byref(img), None, ctypes.byref(dq)) == 0
    dq.data = 1 << 20
    # pad 5 is supported (R22) but needs a descriptor of w + 5 columns: the pad = Hp one is a SHAPE error
    assert L.lib.fht_quadrant(ctypes.byref(img), 0, 5, ctypes.byref(dq), None, 1 << 24, ws_n, None, None) == -3
    ds = L.FhtHough.from_buffer_copy(d)
    ds.shifted = 1
    d3 = L.FhtHough.from_buffer_copy(d)
    d3.data = 1 << 28
    assert L.lib.fhtshift(ctypes.byref(ds), ctypes.byref(d3), None) == -7
    assert L.lib.fhtshift(ctypes.byref(d), ctypes.byref(d), None) == -1                   # aliasing
    big = _img(L, 8192, 8192)
    db = L.FhtHough()
    assert L.lib.fht_hough_describe(1, 0, 0, ctypes.byref(big), None, ctypes.byref(db)) == 0
    db.data = 1 << 40
    assert L.lib.fht_full(ctypes.byref(big), 0, ctypes.byref(db), None, 1 << 44, 1 << 40, None, None) == -5
    # the (out, out_shifted) pair: at least one, no overlap, 16-byte aligned for the TMA row stores
    assert L.lib.fht_full(ctypes.byref(img), 0, None, None, 1 << 24, ws_n, None, None) == -1
    assert L.lib.fht_full(ctypes.byref(img), 0, ctypes.byref(d), ctypes.byref(d), 1 << 24, ws_n, None, None) == -1
    mis = L.FhtHough.from_buffer_copy(d)
    mis.data = (1 << 28) + 4
    assert L.lib.fht_full(ctypes.byref(img), 0, None, ctypes.byref(mis), 1 << 24, ws_n, None, None) == -4
    odd_pitch = L.FhtHough.from_buffer_copy(d)
    odd_pitch.data = 1 << 28
    odd_pitch.row_stride += 1
    odd_pitch.quad_stride = odd_pitch.rows * odd_pitch.row_stride
    odd_pitch.batch_stride = 4 * odd_pitch.quad_stride
    assert L.lib.fht_full(ctypes.byref(img), 0, ctypes.byref(odd_pitch), None, 1 << 24, ws_n, None, None) == -4


def test_status_strings():
    L = _lib()
    for s in range(-8, 1):
        assert L.lib.fht_status_string(s)


def test_cell_segment_matches_oracle():
    """fht_cell_segment (host) == the oracle's §3.2/§3.3 recovery on every cell of small frames:
    QUADRANT (all four), FULL QUADS and CONCAT; count and first/last pixel."""
    from oracle import fht_oracle as O
    L = _lib()
    for h, w in [(4, 4), (5, 7), (8, 3), (6, 6)]:
        img = _img(L, h, w)
        cases = [(L.FHT_MODE_QUADRANT, 0, q) for q in range(4)] + [(L.FHT_MODE_FULL, L.FHT_LAYOUT_QUADS, 0),
                                                                   (L.FHT_MODE_FULL, L.FHT_LAYOUT_CONCAT, 0)]
        for mode, layout, quad in cases:
            d = L.FhtHough()
            assert L.lib.fht_hough_describe(mode, layout, quad, ctypes.byref(img), None, ctypes.byref(d)) == 0
            for slot in range(d.nquad):
                for row in range(d.rows):
                    for col in range(d.cols):
                        sg = L.FhtSegment()
                        assert L.lib.fht_cell_segment(ctypes.byref(d), slot, row, col, ctypes.byref(sg)) == 0
                        if mode == L.FHT_MODE_QUADRANT:
                            q, s, pix = O.cell_segment("quadrant", h, w, row, col, quadrant=quad)
                        else:
                            q, s, pix = O.cell_segment("full", h, w, row, col, quadrant=slot,
                                                       layout="quads" if layout == L.FHT_LAYOUT_QUADS else "concat")
                        assert (sg.quadrant, sg.s, sg.npix) == (q, s, len(pix))
                        if pix:
                            assert (sg.x0, sg.y0, sg.x1, sg.y1) == (*pix[0], *pix[-1])


def test_peaks_and_segment_errors():
    """Synchronous argument checks of the f3 entry points (no device work is enqueued)."""
    L = _lib()
    img = _img(L, 16, 16)
    d = L.FhtHough()
    assert L.lib.fht_hough_describe(L.FHT_MODE_FULL, L.FHT_LAYOUT_QUADS, 0, ctypes.byref(img), None, ctypes.byref(d)) == 0
    d.data = 4096
    n = L.lib.fht_peaks_workspace_bytes(ctypes.byref(d))
    assert n > 0
    ws = 8192
    assert L.lib.fht_peaks(ctypes.byref(d), 0, 4096, 4096, 4096, ws, n, None) == -1       # k < 1
    assert L.lib.fht_peaks(ctypes.byref(d), 33, 4096, 4096, 4096, ws, n, None) == -1      # k > 32
    assert L.lib.fht_peaks(ctypes.byref(d), 8, None, 4096, 4096, ws, n, None) == -1       # NULL output
    assert L.lib.fht_peaks(ctypes.byref(d), 8, 4096, 4096, 4096, ws, n - 1, None) == -6   # workspace too small
    du = L.FhtHough.from_buffer_copy(d)
    du.dtype = L.FHT_U8
    assert L.lib.fht_peaks(ctypes.byref(du), 8, 4096, 4096, 4096, ws, n, None) == -2      # dtype
    sg = L.FhtSegment()
    assert L.lib.fht_cell_segment(ctypes.byref(d), 0, d.rows, 0, ctypes.byref(sg)) == -1  # row out of range
    assert L.lib.fht_cell_segment(ctypes.byref(d), 4, 0, 0, ctypes.byref(sg)) == -1       # slot out of range
    assert L.lib.fht_cell_segment(ctypes.byref(d), 0, 0, d.cols, ctypes.byref(sg)) == -1  # col out of range
    p = L.FhtAnglePlan()
    assert L.lib.fht_angle_plan(16, 16, -15, 15, ctypes.byref(p)) == 0
    dr = L.FhtHough()
    assert L.lib.fht_hough_describe(L.FHT_MODE_RANGE, 0, 0, ctypes.byref(img), ctypes.byref(p), ctypes.byref(dr)) == 0
    assert L.lib.fht_cell_segment(ctypes.byref(dr), 0, 0, 0, ctypes.byref(sg)) == -5      # RANGE: unsupported


def test_pad_describe_and_limits():
    """fht_hough_describe_pad: cols = w_frame + pad; a pad below h_frame - 1 (folding) needs the pad = Hp
    image in the workspace."""
    L = _lib()
    img = _img(L, 100, 60)
    d = L.FhtHough()
    assert L.lib.fht_hough_describe_pad(0, ctypes.byref(img), 99, ctypes.byref(d)) == 0
    assert (d.rows, d.cols) == (128, 60 + 99) and d.row_stride % 4 == 0
    assert L.lib.fht_hough_describe_pad(2, ctypes.byref(img), 59, ctypes.byref(d)) == 0
    assert (d.rows, d.cols) == (64, 100 + 59)
    assert L.lib.fht_hough_describe_pad(0, ctypes.byref(img), -1, ctypes.byref(d)) == 0 and d.cols == 60 + 128
    assert L.lib.fht_hough_describe_pad(0, ctypes.byref(img), -2, ctypes.byref(d)) == -1
    # pads below h_frame - 1 fold: the pad = Hp image (128 x 188 f32, row stride 188) is added to the workspace
    base = L.lib.fht_quadrant_workspace_bytes(ctypes.byref(img), 0, -1)
    assert L.lib.fht_quadrant_workspace_bytes(ctypes.byref(img), 0, 99) == base
    assert L.lib.fht_quadrant_workspace_bytes(ctypes.byref(img), 0, 98) == base + ((128 * 188 * 4 + 255) // 256) * 256


def test_plan_fast_spread_matches_oracle_many():
    """fht_angle_plan's W' (R17) comes from the (min, max) block recursion; the oracle takes the spread
    of e_y - D_s(y) over all (s, y) explicitly. Same W' (and pruned rows) on random shapes and angles,
    non-power-of-two heights included (padding rows hold no pixel)."""
    import random
    from oracle import fht_oracle as O
    L = _lib()
    rnd = random.Random(7)
    for _ in range(60):
        h, w = rnd.randint(1, 300), rnd.randint(4, 300)
        a = rnd.uniform(-85, 80)
        b = rnd.uniform(a + 0.5, min(89, a + 120))
        p = L.FhtAnglePlan()
        r = L.lib.fht_angle_plan(h, w, a, b, ctypes.byref(p))
        try:
            o = O.angle_plan(h, w, a, b)
        except ValueError:
            assert r == -1
            continue
        assert r == 0 and (p.W, p.w_content, p.Hp) == (o.W, o.w_content, o.Hp), (h, w, a, b)
        if math.tan(math.radians(b)) - math.tan(math.radians(a)) <= 1.0:
            assert L.lib.fht_angle_plan_make_pruned(h, w, a, b, ctypes.byref(p)) == 0
            o = O.angle_plan_pruned(h, w, a, b)
            assert (p.W, p.rows) == (o.W, o.rows), (h, w, a, b)


def test_angle_of_row_matches_oracle():
    """fht_angle_of_row (R19) against the oracle's angle_of_row (pinned by the endpoint slopes)."""
    from oracle import fht_oracle as O
    L = _lib()
    for h, w, a, b, flags in [(4096, 4096, -15, 15, 0), (64, 48, 5, 40, 0), (33, 17, -45, 0, 0),
                              (128, 96, -20, 10, 1), (64, 48, -15, 15, 2)]:
        p = L.FhtAnglePlan()
        assert L.lib.fht_angle_plan_make_ex(h, w, a, b, flags, ctypes.byref(p)) == 0
        o = (O.angle_plan_horizontal(h, w, a, b, pruned=bool(flags & 1)) if flags & 2 else
             (O.angle_plan_pruned if flags & 1 else O.angle_plan)(h, w, a, b))
        d = ctypes.c_double()
        for s in sorted({0, 1, p.Hp // 2, p.rows - 1, p.Hp - 1}):
            assert L.lib.fht_angle_of_row(ctypes.byref(p), s, ctypes.byref(d)) == 0
            assert d.value == pytest.approx(O.angle_of_row(s, o), abs=1e-12)
        assert L.lib.fht_angle_of_row(ctypes.byref(p), p.Hp, ctypes.byref(d)) == -1
        assert L.lib.fht_angle_of_row(ctypes.byref(p), -1, ctypes.byref(d)) == -1
    p = L.FhtAnglePlan()
    assert L.lib.fht_angle_plan(256, 256, -15, 15, ctypes.byref(p)) == 0
    d = ctypes.c_double()
    assert L.lib.fht_angle_of_row(ctypes.byref(p), 0, ctypes.byref(d)) == 0 and d.value == pytest.approx(-15, abs=1e-12)
    assert L.lib.fht_angle_of_row(ctypes.byref(p), 255, ctypes.byref(d)) == 0 and d.value == pytest.approx(15, abs=1e-12)


def test_angle_range_by_angles_checks():
    """fht_angle_range(img, theta_min, theta_max, ...) builds the §4 plan itself: its workspace
    size equals fht_workspace_bytes for that plan, and outputs described with another plan, or angle
    errors, are rejected synchronously."""
    L = _lib()
    img = _img(L, 64, 48)
    p = L.FhtAnglePlan()
    assert L.lib.fht_angle_plan(64, 48, -15, 15, ctypes.byref(p)) == 0
    n = L.lib.fht_angle_range_workspace_bytes(ctypes.byref(img), -15.0, 15.0)
    assert n == L.lib.fht_workspace_bytes(L.FHT_MODE_RANGE, ctypes.byref(img), ctypes.byref(p)) and n > 0
    assert L.lib.fht_angle_range_workspace_bytes(ctypes.byref(img), 15.0, -15.0) == 0
    d = L.FhtHough()
    assert L.lib.fht_hough_describe(L.FHT_MODE_RANGE, 0, 0, ctypes.byref(img), ctypes.byref(p), ctypes.byref(d)) == 0
    d.data = 1 << 40
    ws = 1 << 44
    # outputs described for [-15, 15] but the call asks for [-10, 15]
    assert L.lib.fht_angle_range(ctypes.byref(img), -10.0, 15.0, ctypes.byref(d), None, ws, n, None, None) == -3
    assert L.lib.fht_angle_range(ctypes.byref(img), 15.0, -15.0, ctypes.byref(d), None, ws, n, None, None) == -1
    assert L.lib.fht_angle_range(ctypes.byref(img), -15.0, 15.0, None, None, ws, n, None, None) == -1
    assert L.lib.fht_angle_range(ctypes.byref(img), -15.0, 15.0, ctypes.byref(d), None, ws, 16, None, None) == -6


def test_workspace_may_not_alias_image():
    """fht.h: no buffer may overlap another -- a workspace over the image is FHT_ERR_ARG."""
    L = _lib()
    img = _img(L, 64, 64, data=1 << 40)
    d = L.FhtHough()
    assert L.lib.fht_hough_describe(L.FHT_MODE_FULL, 0, 0, ctypes.byref(img), None, ctypes.byref(d)) == 0
    d.data = 1 << 42
    n = L.lib.fht_workspace_bytes(L.FHT_MODE_FULL, ctypes.byref(img), None)
    assert L.lib.fht_full(ctypes.byref(img), 0, ctypes.byref(d), None, (1 << 40) + 64, n, None, None) == -1


@pytest.mark.parametrize("h,w,b,dt", [(1024, 1024, 1, 2), (2048, 2048, 16, 2), (512, 512, 64, 0), (300, 500, 2, 1)])
def test_shard_describe_geometry(h, w, b, dt):
    """fht_shard_describe: S = 2^L / world strips and J = 2^m / world groups per rank,
    chunks of batch * 4 * J * S scratch rows, a band of Hp / world rows starting at rank * Hp / world."""
    L = _lib()
    img = _img(L, h, w, b=b, dt=dt)
    P = 1 << (max(h, w) - 1).bit_length()
    K = P.bit_length() - 1
    Lp = max(K - 6, min(5, (K + 1) // 2))
    mp_ = K - Lp
    for world in (1, 2, 4, 8):
        for rank in range(world):
            sh = L.FhtShard()
            r = L.lib.fht_shard_describe(ctypes.byref(img), world, rank, ctypes.byref(sh))
            if (1 << mp_) % world or (1 << Lp) % world:
                assert r == -5
                continue
            assert r == 0
            assert (sh.m, sh.L, sh.S, sh.J) == (mp_, Lp, (1 << Lp) // world, (1 << mp_) // world)
            assert sh.chunk_rows == b * 4 * sh.J * sh.S
            es = 2 if dt == 0 else 4
            assert sh.scratch_es == es and sh.chunk_bytes == sh.chunk_rows * sh.pitch * es and sh.chunk_bytes % 16 == 0
            assert sh.send_bytes == sh.recv_bytes == world * sh.chunk_bytes
            assert sh.pitch * es % 16 == 0 and sh.pitch >= max(h, w) + (1 << mp_) - 1
            assert (sh.band.nquad, sh.band.rows, sh.band.cols, sh.band.row0) == (4, P // world, 2 * P, rank * P // world)
            assert sh.band.batch == b and sh.band.batch_stride == 4 * sh.band.rows * sh.band.row_stride


def test_shard_describe_errors():
    L = _lib()
    sh = L.FhtShard()
    img = _img(L, 1024, 1024)
    assert L.lib.fht_shard_describe(ctypes.byref(img), 3, 0, ctypes.byref(sh)) == -1       # not a power of two
    assert L.lib.fht_shard_describe(ctypes.byref(img), 2, 2, ctypes.byref(sh)) == -1       # rank out of range
    assert L.lib.fht_shard_describe(ctypes.byref(img), 16, 0, ctypes.byref(sh)) == -5      # > 8 destinations
    assert L.lib.fht_shard_describe(ctypes.byref(_img(L, 512, 1024)), 2, 0, ctypes.byref(sh)) == -5  # not square
    assert L.lib.fht_shard_describe(ctypes.byref(img), 2, 0, None) == -1
    assert L.lib.fht_shard_describe(ctypes.byref(img), 2, 0, ctypes.byref(sh)) == 0
    # pass calls check synchronously: a NULL destination list, a mismatched geometry
    assert L.lib.fht_shard_pass1(ctypes.byref(img), ctypes.byref(sh), None, None) == -1
    other = L.FhtShard()
    assert L.lib.fht_shard_describe(ctypes.byref(_img(L, 2048, 2048)), 2, 0, ctypes.byref(other)) == 0
    assert L.lib.fht_shard_pass2(ctypes.byref(img), ctypes.byref(other), 1 << 40, None, None, None) == -1
