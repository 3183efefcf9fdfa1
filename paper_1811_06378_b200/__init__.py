"""paper_1811_06378_b200 -- B200-native Brady dyadic Fast Hough Transform (arXiv 1811.06378).

Thin torch-facing wrapper over the C ABI of ``libfht.so`` (``include/fht.h``). torch provides
device memory (``data_ptr``) and the current CUDA stream; every step of the transform runs in
the sm_100a kernels behind the ABI. There is no CPU fallback: importing without the built
library, or calling with a non-CUDA tensor, raises.

    full(img, layout="quads", shifted=False, pair=False)   -> HoughImage | (H, S)
    quadrant(img, q, pad=None, shifted=False, pair=False)  -> HoughImage | (H, S)
    angle_plan(h, w, theta_min, theta_max)          -> FhtAnglePlan
    angle_range(img, theta_min, theta_max, shifted=False, pair=False) -> HoughImage | (H, S)
    angle_range(img, plan, ...)                     -> the same for a prepared (pruned / horizontal) plan
    angle_of_row(plan, s)                           -> degrees (R19)
    fhtshift(hough)                                 -> HoughImage

`shifted=True` makes the transform write the fhtshift-ed image directly (fused store);
`pair=True` returns (H, fhtshift(H)) written by the same kernels in one pass.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import (FHT_F32, FHT_I32, FHT_LAYOUT_CONCAT, FHT_LAYOUT_QUADS, FHT_MODE_FULL, FHT_MODE_QUADRANT,
                   FHT_MODE_RANGE, FHT_QA, FHT_QB, FHT_QC, FHT_QD, FHT_U8, FhtAnglePlan, FhtError, FhtHough,
                   FhtImage)

__all__ = ["full", "quadrant", "angle_plan", "angle_range", "angle_of_row", "fhtshift", "full_sharded", "HoughImage",
           "FhtError",
           "QA", "QB", "QC", "QD", "workspace_bytes", "LIB_PATH"]

QA, QB, QC, QD = FHT_QA, FHT_QB, FHT_QC, FHT_QD
LIB_PATH = _lib.LIB_PATH
_DT_IN = {torch.uint8: FHT_U8, torch.int32: FHT_I32, torch.float32: FHT_F32}
_DT_OUT = {FHT_I32: torch.int32, FHT_F32: torch.float32}
_LAYOUTS = {"quads": FHT_LAYOUT_QUADS, "concat": FHT_LAYOUT_CONCAT}


class HoughImage:
    """A Hough image on the device: `storage` is the pitched tensor the kernels wrote,
    `desc` its C descriptor; `view` is the logical [B][nquad][rows][cols] tensor view."""

    def __init__(self, storage: torch.Tensor, desc: FhtHough):
        self.storage = storage
        self.desc = desc
        self.launches = 0  # kernels enqueued by the call that last wrote this image

    @property
    def view(self) -> torch.Tensor:
        d = self.desc
        return self.storage.view(d.batch, d.nquad, d.rows, d.row_stride)[..., : d.cols]

    @property
    def shifted(self) -> bool:
        return bool(self.desc.shifted)

    @property
    def plan(self):
        return self.desc.plan if self.desc.mode == FHT_MODE_RANGE else None


def _image(t: torch.Tensor) -> tuple[FhtImage, torch.Tensor]:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("image must be a CUDA tensor (no CPU path)")
    if t.dtype not in _DT_IN:
        raise TypeError(f"unsupported dtype {t.dtype}; use uint8, int32 or float32")
    if t.dim() == 2:
        t = t.unsqueeze(0)
    if t.dim() != 3:
        raise ValueError("image must be [h][w] or [B][h][w]")
    if t.stride(2) != 1:
        t = t.contiguous()
    img = FhtImage()
    img.data = t.data_ptr()
    img.dtype = _DT_IN[t.dtype]
    img.batch, img.h, img.w = t.shape
    img.batch_stride = t.stride(0) if t.shape[0] > 1 else t.shape[1] * t.stride(1)
    img.row_stride = t.stride(1)
    return img, t


def _alloc_out(mode: int, layout: int, q: int, img: FhtImage, plan, device, pad=None) -> tuple[FhtHough, torch.Tensor]:
    d = FhtHough()
    if pad is not None:
        _lib.check("fht_hough_describe_pad", _lib.lib.fht_hough_describe_pad(q, ctypes.byref(img), pad, ctypes.byref(d)))
    else:
        _lib.check("fht_hough_describe",
                   _lib.lib.fht_hough_describe(mode, layout, q, ctypes.byref(img),
                                               ctypes.byref(plan) if plan is not None else None, ctypes.byref(d)))
    storage = torch.empty(d.batch * d.batch_stride, dtype=_DT_OUT[d.dtype], device=device)
    d.data = storage.data_ptr()
    return d, storage


def workspace_bytes(mode: int, img: FhtImage, plan=None) -> int:
    return int(_lib.lib.fht_workspace_bytes(mode, ctypes.byref(img), ctypes.byref(plan) if plan is not None else None))


def _workspace(nbytes: int, device, workspace: torch.Tensor | None):
    if workspace is not None:
        if workspace.numel() * workspace.element_size() < nbytes:
            raise ValueError("workspace too small")
        return workspace
    return torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)


def _stream(t: torch.Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _descs(kind, img, plan, q, layout, device, shifted, pair, out, out_shifted, pad=None):
    """The (plain, shifted) output pair a transform call writes; None where not requested."""
    want_plain = pair or not shifted
    want_shift = pair or shifted
    res = []
    for want, given in ((want_plain, out), (want_shift, out_shifted)):
        if not want:
            res.append(None)
            continue
        if given is None:
            d, storage = _alloc_out(kind, layout, q, img, plan, device, pad)
            given = HoughImage(storage, d)
        res.append(given)
    return res


def _ptr(h):
    return ctypes.byref(h.desc) if h is not None else None


def _opts(events=None, aux_stream=None):
    """fht_exec_opts for timing events (recorded torch.cuda.Event) and/or an auxiliary
    torch.cuda.Stream for the pass-1 / pass-2 overlap of batched calls; None if neither."""
    if not events and aux_stream is None:
        return None
    o = _lib.FhtExecOpts()
    if events:
        arr = (ctypes.c_void_p * len(events))(*[ctypes.c_void_p(e.cuda_event) for e in events])
        o.events = ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p))
        o.n_events = len(events)
        o._keep = arr
    if aux_stream is not None:
        o.aux_stream = aux_stream.cuda_stream
    return ctypes.byref(o)


def _finish(res, n, shifted, pair):
    for h in res:
        if h is not None:
            h.launches = n
    if pair:
        return res[0], res[1]
    return res[1] if shifted else res[0]


def quadrant(t: torch.Tensor, q: int, pad: int | None = None, shifted: bool = False, pair: bool = False,
             workspace: torch.Tensor | None = None, out: HoughImage | None = None,
             out_shifted: HoughImage | None = None, events=None, aux_stream=None):
    """One quadrant. pad: extension columns (None = Hp; smaller than h_frame - 1 folds lines).
    shifted=True returns fhtshift(H) written directly by the transform; pair=True returns
    (H, fhtshift(H)) from one pass."""
    img, t = _image(t)
    res = _descs(FHT_MODE_QUADRANT, img, None, q, 0, t.device, shifted, pair, out, out_shifted, pad)
    ws_n = int(_lib.lib.fht_quadrant_workspace_bytes(ctypes.byref(img), q, -1 if pad is None else pad))
    ws = _workspace(ws_n, t.device, workspace)
    n = _lib.check("fht_quadrant", _lib.lib.fht_quadrant(ctypes.byref(img), q, -1 if pad is None else pad,
                                                          _ptr(res[0]), _ptr(res[1]), ws.data_ptr(), ws_n,
                                                          _stream(t), _opts(events, aux_stream)))
    return _finish(res, n, shifted, pair)


def full(t: torch.Tensor, layout: str = "quads", shifted: bool = False, pair: bool = False,
         workspace: torch.Tensor | None = None, out: HoughImage | None = None,
         out_shifted: HoughImage | None = None, events=None, aux_stream=None):
    """Full four-quadrant transform. See quadrant() for shifted / pair."""
    img, t = _image(t)
    lay = _LAYOUTS[layout]
    res = _descs(FHT_MODE_FULL, img, None, 0, lay, t.device, shifted, pair, out, out_shifted)
    ws_n = workspace_bytes(FHT_MODE_FULL, img)
    ws = _workspace(ws_n, t.device, workspace)
    n = _lib.check("fht_full", _lib.lib.fht_full(ctypes.byref(img), lay, _ptr(res[0]), _ptr(res[1]),
                                                  ws.data_ptr(), ws_n, _stream(t), _opts(events, aux_stream)))
    return _finish(res, n, shifted, pair)


def angle_plan(h: int, w: int, theta_min_deg: float, theta_max_deg: float, pruned: bool = False,
               horizontal: bool = False) -> FhtAnglePlan:
    """§4 plan (scale + shear, all Hp rows); pruned=True: the shift-range-pruned plan (shear only,
    rows s <= S_max); horizontal=True: angles from the horizontal, the plan built on
    the transposed image (mostly-horizontal lines, f4)."""
    p = FhtAnglePlan()
    flags = (_lib.FHT_PLAN_PRUNED if pruned else 0) | (_lib.FHT_PLAN_HORIZONTAL if horizontal else 0)
    _lib.check("fht_angle_plan_make_ex", _lib.lib.fht_angle_plan_make_ex(h, w, float(theta_min_deg),
                                                                          float(theta_max_deg), flags, ctypes.byref(p)))
    return p


def angle_of_row(plan: FhtAnglePlan, s: int) -> float:
    """Inclination (degrees) of the lines row s of a range output holds (R19)."""
    d = ctypes.c_double()
    _lib.check("fht_angle_of_row", _lib.lib.fht_angle_of_row(ctypes.byref(plan), int(s), ctypes.byref(d)))
    return d.value


def angle_range(t: torch.Tensor, theta_min, theta_max: float | None = None, shifted: bool = False,
                pair: bool = False, workspace: torch.Tensor | None = None, out: HoughImage | None = None,
                out_shifted: HoughImage | None = None, events=None, aux_stream=None):
    """Angle-range-restricted transform (§4, "a transform for an arbitrary range of angles";
    P:146-152): `angle_range(t, theta_min, theta_max)` calls fht_angle_range, which builds the §4 plan
    itself; `angle_range(t, plan)` calls fht_angle_range_plan with a prepared plan (pruned or
    mostly-horizontal plans). See quadrant() for shifted / pair."""
    img, t = _image(t)
    by_angles = not isinstance(theta_min, FhtAnglePlan)
    plan = None if by_angles else theta_min
    need_out = ((pair or not shifted) and out is None) or ((pair or shifted) and out_shifted is None)
    if by_angles and need_out:  # the plan only describes outputs the caller did not pass
        plan = angle_plan(int(img.h), int(img.w), float(theta_min), float(theta_max))
    res = _descs(FHT_MODE_RANGE, img, plan, 0, 0, t.device, shifted, pair, out, out_shifted)
    if by_angles:
        ws_n = (workspace.numel() * workspace.element_size() if workspace is not None else
                int(_lib.lib.fht_angle_range_workspace_bytes(ctypes.byref(img), float(theta_min), float(theta_max))))
        ws = _workspace(ws_n, t.device, workspace)
        n = _lib.check("fht_angle_range", _lib.lib.fht_angle_range(
            ctypes.byref(img), float(theta_min), float(theta_max), _ptr(res[0]), _ptr(res[1]), ws.data_ptr(), ws_n,
            _stream(t), _opts(events, aux_stream)))
    else:
        ws_n = workspace_bytes(FHT_MODE_RANGE, img, plan)
        ws = _workspace(ws_n, t.device, workspace)
        n = _lib.check("fht_angle_range_plan", _lib.lib.fht_angle_range_plan(
            ctypes.byref(img), ctypes.byref(plan), _ptr(res[0]), _ptr(res[1]), ws.data_ptr(), ws_n, _stream(t),
            _opts(events, aux_stream)))
    return _finish(res, n, shifted, pair)


def fhtshift(h: HoughImage, out: HoughImage | None = None) -> HoughImage:
    if out is None:
        d = FhtHough.from_buffer_copy(h.desc)
        storage = torch.empty_like(h.storage)
        d.data = storage.data_ptr()
        out = HoughImage(storage, d)
    out.desc.shifted = 0
    out.launches = _lib.check("fhtshift", _lib.lib.fhtshift(ctypes.byref(h.desc), ctypes.byref(out.desc), _stream(h.storage)))
    return out


def peaks(h: HoughImage, k: int = 16, workspace: torch.Tensor | None = None):
    """Top-k peaks of every Hough plane (DESIGN R25): (values, rows, cols), each
    [batch][nquad][k] on the device; missing peaks have row = col = -1."""
    d = h.desc
    shape = (d.batch, d.nquad, k)
    vals = torch.empty(shape, dtype=h.storage.dtype, device=h.storage.device)
    rows = torch.empty(shape, dtype=torch.int32, device=h.storage.device)
    cols = torch.empty(shape, dtype=torch.int32, device=h.storage.device)
    ws_n = _lib.lib.fht_peaks_workspace_bytes(ctypes.byref(d))
    ws = _workspace(ws_n, h.storage.device, workspace)
    _lib.check("fht_peaks", _lib.lib.fht_peaks(ctypes.byref(d), int(k), vals.data_ptr(), rows.data_ptr(),
                                                 cols.data_ptr(), ws.data_ptr(), ws_n, _stream(h.storage)))
    return vals, rows, cols


def cell_segment(h: HoughImage, row: int, col: int, slot: int = 0) -> dict | None:
    """The pattern of Hough cell (row, col) on the original image (CONCAT rows by P:111-113):
    {"quadrant", "s", "npix", "first": (x, y), "last": (x, y)}, or None in the black zone."""
    sg = _lib.FhtSegment()
    _lib.check("fht_cell_segment", _lib.lib.fht_cell_segment(ctypes.byref(h.desc), int(slot), int(row), int(col),
                                                               ctypes.byref(sg)))
    if sg.npix == 0:
        return None
    return {"quadrant": sg.quadrant, "s": sg.s, "npix": sg.npix, "first": (sg.x0, sg.y0), "last": (sg.x1, sg.y1)}


class Graph:
    """A CUDA graph of one call sequence through this library (torch.cuda.CUDAGraph): `fn` is run
    once eagerly (one-time attributes, tensor maps), then captured on a side stream and replayed by
    `replay()` -- one host launch instead of the per-call descriptor checks, tensor-map encodes and
    kernel launches. Every buffer `fn` uses (input, outputs, workspace) must be preallocated and stay
    alive; the library's launches (programmatic dependent launch, the auxiliary-stream fork/join via
    events) are captured as graph edges.

        g = fht.Graph(lambda: fht.full(t, pair=True, out=h, out_shifted=s, workspace=ws))
        g.replay()
    """

    def __init__(self, fn):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.result = fn()

    def replay(self):
        self.graph.replay()
        return self.result


from .sharding import full_sharded, shard_describe  # noqa: E402  (one image over several GPUs)
