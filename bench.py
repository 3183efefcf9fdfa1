#!/usr/bin/env python
"""Benchmark of the B200 FHT hot path (BASELINE.json metric: input Gpixel/s for the full
four-quadrant FHT; achieved HBM GB/s vs roofline).

    python bench.py [--gpus N --steps K --warmup W] [--config 5|2|3|4|1] [--impl ours|reference]

A step = one pass of the config's whole hot path over one batch of synthetic input already
resident in HBM:
  C5 (default: the largest full-FHT config, whose 4.6 GB working set is far beyond L2, so the line
      measures HBM): full four-quadrant FHT of 16 x 2048^2 f32 images, writing the four Hough
      quadrants AND their fhtshift regrouping (both outputs, one pass); the single-destination step
      (only the fhtshift-ed image, BASELINE.md's compulsory bytes) is reported beside it;
  C2: the same on one 1024^2 image; C3: full FHT of 64 x 512^2 u8 (int32 out); C4: angle-range FHT
      [-15, 15] deg of 4096^2 f32 + fhtshift; C1: one quadrant of a 256^2 u8 image.
Rank 0 prints ONE JSON line. Under torchrun every rank transforms its own batch (weak scaling,
no data-path collective: the images are independent); the step time is the max
over ranks. The other configs are timed too and reported under "configs" (not the headline).

--impl reference runs the oracle (oracle/fht_oracle.py, tier-2 numpy recursion, float64/int64)
on the host cores over a bounded sample of the same workload: the task's reference arm.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input Gpixel/s for full 4-quadrant FHT; achieved HBM GB/s vs roofline"
L2_FLUSH_BYTES = 512 << 20
TARGET_FRAC_8TBS = 0.60   # north_star: >= 60% of the compulsory-byte roofline at 8 TB/s


def l2_bytes(dev) -> int:
    """The device's L2 size (cudaDevAttrL2CacheSize through torch)."""
    import torch
    return int(torch.cuda.get_device_properties(dev).L2_cache_size)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured: MEASURED_PEAKS.json hbm_gbs (copy, read+write bytes)"
    return 6650.0, "fallback: B200_PROFILING.md 6.65 TB/s"


def load_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu --set full
    capture (profiles/ncu_traffic.json, written by tools/ncu_summary.py), or {}."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    return json.load(open(p)) if os.path.exists(p) else {}


# ----------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """Polls NVML (SM clock, max clock, clock-event reasons) from a thread while active."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index, self.samples, self.stop = index, [], threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001 -- no NVML: report unsampled
            pass

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = (nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                      if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons")
                      else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h))
                self.samples.append((sm, rs))
            except Exception:  # noqa: BLE001
                return
            time.sleep(0.0005)

    def __enter__(self):
        if self.ok:
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
            time.sleep(0.002)
        return self

    def __exit__(self, *a):
        if self.ok:
            time.sleep(0.002)
            self.stop.set()
            self.thread.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({n for _, rs in self.samples for n, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "NVML polled during the timed region"}


# ----------------------------------------------------------------------------------------- workloads
def pow2(n):
    return 1 << (n - 1).bit_length()


def geometry(cfg_id, c):
    """Algorithmic bytes: input read once, every output written once."""
    B, h, w = c["batch"], c["h"], c["w"]
    in_b = B * h * w * (1 if c["dtype"] == "u8" else 4)
    Hp, Wp = pow2(h), pow2(w)
    if c["mode"] == "quadrant":
        cells = B * Hp * (w + Hp)
        ndest = 1
    elif c["mode"] == "full":
        cells = B * 4 * max(Hp, Wp) * (Hp + Wp)
        ndest = 2 if cfg_id in (2, 5) else 1
    else:
        cells = None  # range: from the plan (filled in by the caller)
        ndest = 2
    return in_b, cells, ndest


def make_step(fht, cfg_id, c, t, outs, plan=None, aux=None, single=False):
    """step(events=None) -> kernel launches enqueued (all through the C ABI). `aux`: the second
    stream on which batched calls overlap pass 1 of the next chunk with pass 2 (not used while
    per-kernel events are recorded). `single`: C2/C5 write only the fhtshift-ed image."""
    if c["mode"] == "quadrant":
        def step(events=None):
            outs["h"] = fht.quadrant(t, fht.QA, out=outs.get("h"), workspace=outs.get("ws"), events=events)
            return outs["h"].launches
        return step
    if c["mode"] == "full":
        pair = cfg_id in (2, 5) and not single

        def step(events=None):
            a = None if events else aux
            if single:
                outs["s"] = fht.full(t, shifted=True, out_shifted=outs.get("s"), workspace=outs.get("ws"),
                                     events=events, aux_stream=a)
                return outs["s"].launches
            if pair:
                outs["h"], outs["s"] = fht.full(t, pair=True, out=outs.get("h"), out_shifted=outs.get("s"),
                                                workspace=outs.get("ws"), events=events, aux_stream=a)
            else:
                outs["h"] = fht.full(t, out=outs.get("h"), workspace=outs.get("ws"), events=events, aux_stream=a)
            return outs["h"].launches
        return step

    def step(events=None):  # fht_angle_range(img, theta_min, theta_max): the §4 plan is built inside the call
        outs["h"], outs["s"] = fht.angle_range(t, c["theta_min"], c["theta_max"], pair=True, out=outs.get("h"),
                                               out_shifted=outs.get("s"), workspace=outs.get("ws"), events=events)
        return outs["h"].launches
    return step


# ----------------------------------------------------------------------------------------- oracle arm
_ORACLE_IMGS = None


def _oracle_unit(args):
    cfg_id, b, q = args
    import synth
    from oracle import fht_oracle as O
    img = _ORACLE_IMGS[b]
    c = synth.CONFIGS[cfg_id]
    if c["mode"] == "range":
        p = O.angle_plan(c["h"], c["w"], c["theta_min"], c["theta_max"])
        R = O.angle_range(img, p)
        O.fhtshift_range(R, p)
    elif c["mode"] == "quadrant":
        O.hough_recursive(img, O.QA)
    else:
        Hp, Wp = O.full_padding(*img.shape)
        fr = O.quadrant_frame(img, q, square_to=(Hp, Wp))
        H = O.hough_of_frame_recursive(fr)
        if cfg_id in (2, 5):
            O.fhtshift_quadrant(H, fr.sigma)
    return 0


def oracle_sample(cfg_id: int, c, imgs, min_seconds: float = 10.0, max_units: int = 4096):
    """Time the oracle as it stands (tier-2 recursion, float64/int64) on the host cores over a
    bounded sample of the workload: whole (image, quadrant) units, repeated round-robin over the
    batch until >= min_seconds of wall time, in a fork pool (one process per core)."""
    global _ORACLE_IMGS
    _ORACLE_IMGS = imgs
    if c["mode"] == "full":
        base = [(cfg_id, b, q) for b in range(imgs.shape[0]) for q in range(4)]
        per_unit_px = c["h"] * c["w"] / 4.0
    else:
        base = [(cfg_id, 0, 0)]
        per_unit_px = c["h"] * c["w"]
    cores = max(1, len(os.sched_getaffinity(0)))
    done, t_total = 0, 0.0
    with mp.get_context("fork").Pool(cores) as pool:
        while t_total < min_seconds and done < max_units:
            batch = [base[(done + i) % len(base)] for i in range(max(cores, 1))]
            t0 = time.perf_counter()
            pool.map(_oracle_unit, batch, chunksize=1)
            t_total += time.perf_counter() - t0
            done += len(batch)
    px = per_unit_px * done
    kind = {"full": "full FHT", "quadrant": "one quadrant", "range": "angle-range FHT"}[c["mode"]]
    return {"value": px / t_total / 1e9, "unit": "Gpixel/s", "cores": cores, "kind": "oracle",
            "sample": f"{done} (image, quadrant) units of {c['name']} ({kind}"
                      f"{' + fhtshift' if cfg_id in (2, 4, 5) else ''}); oracle tier-2 numpy recursion, "
                      f"float64/int64, one process per core, {t_total:.1f} s wall"}


# ----------------------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-shift-bench", action="store_true", help="skip the standalone fhtshift (SURVEY a7) lines")
    ap.add_argument("--no-graph", action="store_true", help="C1/C2 headline with eager calls instead of graph replay")
    ap.add_argument("--no-aux", action="store_true",
                    help="no auxiliary stream (one stream, merged 4-slot launches: what the per-kernel loop runs)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--extra-configs", default="2,3,4,1",
                    help="other configs also timed (reported under 'configs', not the headline)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    import synth
    c = synth.CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        imgs = synth.batch(args.config)
        per_step = max(2.0, min(20.0, 150.0 / (args.steps + args.warmup)))
        vals, last = [], None
        for i in range(args.warmup + args.steps):
            last = oracle_sample(args.config, c, imgs, min_seconds=per_step)
            if i >= args.warmup:
                vals.append(last["value"])
        v = statistics.mean(vals)
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Gpixel/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64" if c["dtype"] == "f32" else "int64", "data": "synthetic",
                "config": {"workload": c["name"], "batch": c["batch"], "h": c["h"], "w": c["w"]},
                "cpu_baseline": dict(last, value=v),
                "e2e": {"value": v, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    import paper_1811_06378_b200 as fht

    peak_gbs, peak_src = load_peaks()
    traffic = load_traffic()

    def barrier():
        if world > 1:
            dist.barrier()

    from paper_1811_06378_b200.sharding import max_over_ranks as _mor, rank_images

    def max_over_ranks(x):
        return _mor(x, device=dev)

    L2_BYTES = l2_bytes(dev)

    def run_config(cfg_id, steps, warmup, with_e2e, use_graph=True, single=False):
        cc = synth.CONFIGS[cfg_id]
        mine = rank_images(cc["batch"], rank, world)  # weak scaling: this rank's own images
        imgs = synth.batch(cfg_id, first=mine.start)
        t = torch.from_numpy(imgs).to(dev)
        in_b, cells, ndest = geometry(cfg_id, cc)
        if single:
            ndest = 1
        plan = None
        if cc["mode"] == "range":
            plan = fht.angle_plan(cc["h"], cc["w"], cc["theta_min"], cc["theta_max"])
            cells = cc["batch"] * plan.Hp * plan.W
        out_b = cells * 4 * ndest
        outs = {}
        aux = None if args.no_aux else torch.cuda.Stream(device=dev)
        step = make_step(fht, cfg_id, cc, t, outs, plan, aux, single=single)
        # kernels per step as the per-kernel breakdown (below) launches them: with events the
        # library runs every call on the launching stream (a single-image full transform otherwise
        # splits its two orientations over the main and auxiliary streams, 4 launches instead of 2)
        probe = torch.cuda.Event(enable_timing=True)
        probe.record()
        n_launch = step(events=[probe])
        torch.cuda.synchronize()
        ws_bytes = 0
        flush = None
        if in_b + out_b < 2 * L2_BYTES:
            flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
        stream = torch.cuda.current_stream()
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        # C1/C2 headline steps are CUDA-graph replays of the same call (one host launch
        # per step instead of ~40 us of descriptor checks, tensor-map encodes and launches); stated in
        # config.timing. Batched configs are GPU-bound and run the eager call.
        graph = None
        if use_graph and cfg_id in (1, 2):
            outs["ws"] = torch.empty(max(1, fht.workspace_bytes(
                {"quadrant": fht.FHT_MODE_QUADRANT, "full": fht.FHT_MODE_FULL, "range": fht.FHT_MODE_RANGE}[cc["mode"]],
                fht._image(t)[0], plan)), dtype=torch.uint8, device=dev)
            graph = fht.Graph(step)
            for _ in range(warmup):
                graph.replay()
            torch.cuda.synchronize()
        launches_eager = step()
        torch.cuda.synchronize()
        # per-step events: [0] before the first kernel ... [n_launch] after the last (fht_exec_opts)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n_launch + 1)] for _ in range(steps)]
        for row in evs:  # materialise the cudaEvent_t handles
            for e in row:
                e.record(stream)
        torch.cuda.synchronize()
        # (1) headline: events only around each step (nothing between the kernels, so the
        # programmatic dependent launch between pass 1 and pass 2 keeps its overlap)
        s0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        s1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        launches = 0
        barrier()
        torch.cuda.synchronize()
        with ClockSampler(local_rank) as clk:
            t_wall = time.perf_counter()
            for i in range(steps):
                if flush is not None:
                    flush.zero_()
                s0[i].record(stream)
                if graph is not None:
                    graph.replay()
                    launches += launches_eager
                else:
                    launches += step()
                s1[i].record(stream)
            torch.cuda.synchronize()
            t_wall = time.perf_counter() - t_wall
        barrier()
        step_ms = [s0[i].elapsed_time(s1[i]) for i in range(steps)]
        ms = max_over_ranks(statistics.mean(step_ms))
        # (2) per-kernel breakdown for the roofline: the same K steps again with an event recorded
        # by the library before / after every kernel (fht_exec_opts) on the launching stream
        for i in range(steps):
            if flush is not None:
                flush.zero_()
            step(events=evs[i])
        torch.cuda.synchronize()
        ker_ms = [[evs[i][k].elapsed_time(evs[i][k + 1]) for i in range(steps)] for k in range(n_launch)]
        kms = [max_over_ranks(statistics.mean(x)) for x in ker_ms]
        px = cc["batch"] * cc["h"] * cc["w"]
        res = {"workload": cc["name"], "ms_per_step": ms, "gpix_s": px * world / (ms * 1e-3) / 1e9,
               "in_bytes": in_b, "out_bytes": out_b, "launches_per_step": launches // steps,
               "l2": "flushed between steps (512 MiB write outside the step events)" if flush is not None
               else "working set > L2 (no flush needed)",
               "clocks": clk.summary(), "wall_s": t_wall, "graph": graph is not None}
        res["step_gbs"] = (in_b + out_b) / (ms * 1e-3) / 1e9
        # launch order: [range tables,] then (pass 1, pass 2) per batch chunk / orientation -- or ONE
        # k_pipe launch (both passes in one persistent kernel, fht_pipe.cuh) for the pipelined frames
        first = 1 if cc["mode"] == "range" else 0
        if n_launch - first == 1:
            names = ["k_pipe"]
        else:
            # pass 1 of 64-row strips of 4-byte images (Hp >= 2048; full mode, or the §4 range loader) is the persistent kernel k_p1p
            hp = 1 << (max(cc["h"], 1) - 1).bit_length()
            p1n = ("k_p1p" if cc["mode"] in ("full", "range") and cc["dtype"] in ("f32", "i32") and hp >= 2048 and cc["w"] % 32 == 0
                   and os.environ.get("FHT_P1_PERSIST", "1") != "0" else "k_p1")
            if (cc["dtype"] == "u8" and hp in (256, 512) and cc["w"] % 128 == 0 and cc["mode"] in ("full", "quadrant")
                    and os.environ.get("FHT_P1_PERSIST", "1") != "0"):
                p1n = "k_p1p8"  # 16-row strips of u8 images: the persistent u8 kernel
            names = (["k_range_tables"] if first else []) + [p1n, "k_p2"] * ((n_launch - first) // 2)
        p2 = [k for k in range(n_launch) if names[k] == "k_p2"]
        p2_ms = sum(kms[k] for k in p2)
        p1_ms = sum(kms[k] for k in range(n_launch) if names[k] in ("k_p1", "k_p1p", "k_p1p8", "k_range_tables"))
        pipe_ms = sum(kms[k] for k in range(n_launch) if names[k] == "k_pipe")
        tot = sum(kms)
        # the dominant kernel: k_pipe (one read of the image + every output written, per launch) or
        # pass 2 (every output written; per-launch algorithmic bytes, several pairs with chunking).
        # Its share of the step's kernel time comes from the same per-kernel loop.
        if pipe_ms:
            dom = {"kernel": "k_pipe (both passes: image -> L2-resident scratch ring -> Hough image [+ fhtshift])",
                   "ms": pipe_ms, "launches": 1, "alg_bytes": in_b + out_b}
        else:
            dom = {"kernel": "k_p2 (pass 2: levels m+1..K, scratch -> Hough image [+ fhtshift])",
                   "ms": p2_ms, "launches": len(p2), "alg_bytes": out_b}
        res["kernels"] = {"names": names, "ms": kms, "pass1_ms": p1_ms, "pass2_ms": p2_ms, "pipe_ms": pipe_ms,
                          "pass2_launches": len(p2), "dominant": dom["kernel"],
                          "dominant_share_of_step": dom["ms"] / tot if tot else None}
        res["dominant"] = dom
        res["pass2_gbs"] = dom["alg_bytes"] / (dom["ms"] * 1e-3) / 1e9
        if with_e2e:
            res["e2e"] = e2e_config(cfg_id, cc, imgs, plan, min(steps, 10) if in_b + out_b > (1 << 30) else steps, px)
        del outs, t, flush
        torch.cuda.empty_cache()
        return res

    def e2e_config(cfg_id, cc, imgs, plan, steps, px):
        """Same metric through the public API with the input in pinned host memory and the step's
        result(s) read back to pinned host memory, every step's copies inside the timed region.
        Two slots pipeline consecutive steps: step i+1's upload and transform (compute stream)
        overlap step i's download (copy stream; the opposite copy direction)."""
        pinned_in = torch.from_numpy(imgs).pin_memory()
        comp = torch.cuda.Stream(device=dev)
        down = torch.cuda.Stream(device=dev)
        slots = []
        # two slots pipeline consecutive steps; under torchrun one slot per rank (the pinned host buffers of
        # C5's 4.3 GB of outputs per slot would be multiplied by every rank on the node)
        for _ in range(2 if world == 1 else 1):
            t_dev = torch.empty(pinned_in.shape, dtype=pinned_in.dtype, device=dev)
            outs = {}
            slots.append({"t": t_dev, "outs": outs, "step": make_step(fht, cfg_id, cc, t_dev, outs, plan),
                          "host": {}, "done": torch.cuda.Event(), "free": torch.cuda.Event()})

        def run(i):
            sl = slots[i % len(slots)]
            with torch.cuda.stream(comp):
                comp.wait_event(sl["free"])            # this slot's previous download has finished
                sl["t"].copy_(pinned_in, non_blocking=True)
                sl["step"]()
                sl["done"].record(comp)
            d2h = 0
            with torch.cuda.stream(down):
                down.wait_event(sl["done"])
                for k in ("h", "s"):
                    if k in sl["outs"]:
                        st = sl["outs"][k].storage
                        if k not in sl["host"]:
                            sl["host"][k] = torch.empty(st.shape, dtype=st.dtype).pin_memory()
                        sl["host"][k].copy_(st, non_blocking=True)
                        d2h += sl["host"][k].numel() * 4
                sl["free"].record(down)
            return pinned_in.numel() * pinned_in.element_size(), d2h
        for sl in slots:
            sl["free"].record(down)
        for i in range(4):
            run(i)
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(comp)
        down.wait_stream(comp)
        for i in range(steps):
            hb, db = run(i)
        comp.wait_stream(down)
        t1.record(comp)
        torch.cuda.synchronize()
        ms = max_over_ranks(t0.elapsed_time(t1) / steps)
        return {"value": px * world / (ms * 1e-3) / 1e9, "unit": "Gpixel/s", "h2d_bytes_per_step": hb,
                "d2h_bytes_per_step": db, "ms_per_step": ms,
                "pipeline": ("two slots: upload + transform of step i+1 overlap the download of step i" if len(slots) == 2
                             else "one slot per rank (torchrun): upload, transform, download in sequence")}

    def shift_standalone(cfg_id, steps=20):
        """SURVEY a7 standalone fhtshift (one warp per row, 16-byte rotation) on the config's Hough
        image: read + write of every cell; working set > L2 for C5 (no flush needed)."""
        cc = synth.CONFIGS[cfg_id]
        t_in = torch.from_numpy(synth.batch(cfg_id)).to(dev)
        if cc["mode"] == "range":
            h = fht.angle_range(t_in, fht.angle_plan(cc["h"], cc["w"], cc["theta_min"], cc["theta_max"]))
        else:
            h = fht.full(t_in)
        del t_in
        out = fht.fhtshift(h)
        for _ in range(3):
            fht.fhtshift(h, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fht.fhtshift(h, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        nbytes = 2 * h.storage.numel() * h.storage.element_size()
        res = {"workload": cc["name"], "mode": cc["mode"], "bytes_per_call": nbytes, "ms_per_call": ms,
               "achieved_gbs": nbytes / (ms * 1e-3) / 1e9, "peak_gbs": peak_gbs,
               "frac": nbytes / (ms * 1e-3) / 1e9 / peak_gbs, "launches_per_call": out.launches}
        del h, out
        torch.cuda.empty_cache()
        return res

    def range_pruned(steps=20):
        """SURVEY §8(f) f2 on config 4's image: shear-only plan, rows s <= S_max only (2196 of 4096 for
        [-15, 15]); the Hough rows and their fhtshift written in one pass, as config 4 does."""
        cc = synth.CONFIGS[4]
        t_in = torch.from_numpy(synth.batch(4)).to(dev)
        plan = fht.angle_plan(cc["h"], cc["w"], cc["theta_min"], cc["theta_max"], pruned=True)
        outs = {}

        def step():
            outs["h"], outs["s"] = fht.angle_range(t_in, plan, pair=True, out=outs.get("h"), out_shifted=outs.get("s"))
            return outs["h"].launches
        n = step()
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        nbytes = t_in.numel() * 4 + 2 * plan.rows * plan.W * 4
        res = {"workload": "c4_range_pruned_f32_4096", "rows": plan.rows, "W": plan.W, "ms_per_step": ms,
               "gpix_s": cc["h"] * cc["w"] / (ms * 1e-3) / 1e9, "compulsory_bytes": nbytes,
               "step_gbs": nbytes / (ms * 1e-3) / 1e9, "step_frac_of_measured_hbm": nbytes / (ms * 1e-3) / 1e9 / peak_gbs,
               "launches_per_step": n, "l2": "working set > L2 (no flush needed)"}
        del t_in, outs
        torch.cuda.empty_cache()
        return res

    def peaks_bench(steps=20, k=16):
        """top-k peaks of config 3's Hough output (64 images x 4 quadrants of
        512 x 1024 i32); algorithmic bytes = one read of every plane."""
        t_in = torch.from_numpy(synth.batch(3)).to(dev)
        h = fht.full(t_in)
        del t_in
        out = fht.peaks(h, k)
        for _ in range(3):
            out = fht.peaks(h, k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            out = fht.peaks(h, k)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        nbytes = h.storage.numel() * 4
        res = {"workload": "c3 Hough planes, top-16 peaks per plane", "planes": int(h.desc.batch * h.desc.nquad),
               "k": k, "ms_per_call": ms, "bytes_per_call": nbytes, "achieved_gbs": nbytes / (ms * 1e-3) / 1e9,
               "frac_of_measured_hbm": nbytes / (ms * 1e-3) / 1e9 / peak_gbs, "launches_per_call": 2,
               "l2": "working set 537 MB > L2 (no flush needed)"}
        del h, out
        torch.cuda.empty_cache()
        return res

    def back_to_back(cfg_id, steps=200):
        """Steps issued back to back (no L2 flush, so the input may stay in L2: informational, not the
        headline): wall time per step with the eager Python/C call vs a CUDA-graph replay of the same
        call -- shows whether the host keeps ahead of the GPU."""
        import time as _t
        cc = synth.CONFIGS[cfg_id]
        t_in = torch.from_numpy(synth.batch(cfg_id)).to(dev)
        outs = {}
        aux = torch.cuda.Stream(device=dev)
        plan = fht.angle_plan(cc["h"], cc["w"], cc["theta_min"], cc["theta_max"]) if cc["mode"] == "range" else None
        step = make_step(fht, cfg_id, cc, t_in, outs, plan, aux)
        step()
        outs["ws"] = torch.empty(max(1, fht.workspace_bytes(
            {"quadrant": fht.FHT_MODE_QUADRANT, "full": fht.FHT_MODE_FULL, "range": fht.FHT_MODE_RANGE}[cc["mode"]],
            fht._image(t_in)[0], plan)), dtype=torch.uint8, device=dev)
        res = {"workload": cc["name"], "steps": steps, "l2": "not flushed (back to back)"}
        for label, run in (("eager", None), ("graph", fht.Graph(step))):
            go = step if run is None else run.replay
            for _ in range(10):
                go()
            torch.cuda.synchronize()
            w0 = _t.perf_counter()
            for _ in range(steps):
                go()
            h_us = (_t.perf_counter() - w0) / steps * 1e6
            torch.cuda.synchronize()
            res[label] = {"wall_us_per_step": (_t.perf_counter() - w0) / steps * 1e6, "host_us_per_step": h_us}
        del t_in, outs
        torch.cuda.empty_cache()
        return res

    head = run_config(args.config, args.steps, args.warmup, with_e2e=True, use_graph=not args.no_graph)
    single_line = None
    if args.config in (2, 5):
        # BASELINE.md's compulsory bytes: one read of the image + ONE write of the Hough output -- the
        # step that writes only the fhtshift-ed image (the regrouped Hough image, §5), same kernels
        try:
            sd = run_config(args.config, args.steps, args.warmup, with_e2e=False, use_graph=not args.no_graph,
                            single=True)
            comp = sd["in_bytes"] + sd["out_bytes"]
            single_line = {
                "step": "full 4-quadrant FHT writing only fhtshift(H) (one destination)",
                "ms_per_step": sd["ms_per_step"], "gpix_s": sd["gpix_s"], "compulsory_bytes": comp,
                "step_gbs": sd["step_gbs"], "step_frac_of_measured_hbm": sd["step_gbs"] / peak_gbs,
                "step_frac_of_8tbs": sd["step_gbs"] / 8000.0,
                "target_ms_60pct_of_8tbs": comp / (TARGET_FRAC_8TBS * 8000e9) * 1e3,
                "target_met": sd["step_gbs"] / 8000.0 >= TARGET_FRAC_8TBS,
                "kernels": sd["kernels"], "dominant_frac_of_measured_hbm": sd["pass2_gbs"] / peak_gbs,
                "launches_per_step": sd["launches_per_step"], "clocks": sd["clocks"], "l2": sd["l2"]}
        except Exception as e:  # noqa: BLE001 -- report, do not hide
            single_line = {"error": repr(e)}
    b2b_line = None
    if not args.no_shift_bench:
        try:
            b2b_line = back_to_back(args.config)
        except Exception as e:  # noqa: BLE001 -- report, do not hide
            b2b_line = {"error": repr(e)}
    peaks_line = None
    if not args.no_shift_bench:
        try:
            peaks_line = peaks_bench()
        except Exception as e:  # noqa: BLE001 -- report, do not hide
            peaks_line = {"workload": "c3 peaks", "error": repr(e)}
    pruned_line = None
    if not args.no_shift_bench:
        try:
            pruned_line = range_pruned()
        except Exception as e:  # noqa: BLE001 -- report, do not hide
            pruned_line = {"workload": "c4_range_pruned_f32_4096", "error": repr(e)}
    shift_lines = []
    if not args.no_shift_bench:
        for cid in (5, 4):
            try:
                shift_lines.append(shift_standalone(cid))
            except Exception as e:  # noqa: BLE001 -- report, do not hide
                shift_lines.append({"workload": synth.CONFIGS[cid]["name"], "error": repr(e)})
    extra = {}
    extra_ids = [] if args.extra_configs in ("", "none") else [int(x) for x in args.extra_configs.split(",")]
    for cid in [x for x in extra_ids if x != args.config]:
        try:
            r = run_config(cid, max(5, args.steps // 4), 3, with_e2e=False)
            extra[r["workload"]] = {k: r[k] for k in ("ms_per_step", "gpix_s", "step_gbs", "pass2_gbs", "kernels",
                                                      "launches_per_step", "l2")}
            extra[r["workload"]]["step_frac_of_measured_hbm"] = r["step_gbs"] / peak_gbs
            extra[r["workload"]]["dominant_frac_of_measured_hbm"] = r["pass2_gbs"] / peak_gbs
        except Exception as e:  # noqa: BLE001 -- report, do not hide
            extra[synth.CONFIGS[cid]["name"]] = {"error": repr(e)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = oracle_sample(args.config, c, synth.batch(args.config), min_seconds=args.cpu_seconds)
    tr = traffic.get(c["name"], {}).get(head["dominant"]["kernel"].split()[0])
    line = {
        "metric": METRIC, "value": head["gpix_s"], "unit": "Gpixel/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if c["dtype"] == "f32" else "int32", "data": "synthetic",
        "config": {"workload": c["name"], "batch_per_gpu": c["batch"], "global_batch": c["batch"] * world,
                   "h": c["h"], "w": c["w"],
                   "step": {1: "QA quadrant", 2: "full 4-quadrant FHT + fhtshift (both written)",
                            3: "full 4-quadrant FHT", 4: "angle-range FHT + fhtshift (both written)",
                            5: "full 4-quadrant FHT + fhtshift (both written)"}[args.config],
                   "parallelism": f"dp{world} (independent images per rank, no collective)",
                   "l2": head["l2"],
                   "timing": ("CUDA events on the launching stream around each step (none between its kernels), "
                              "mean over steps; max over ranks; per-kernel times from a second K-step loop of eager "
                              "calls with an event around every kernel"
                              + ("; headline steps are CUDA-graph replays of the same call (SURVEY 8(d): allowed "
                                 "for C1/C2)" if head["graph"] else "; headline steps are eager calls"))},
        "roofline": {"bound": "hbm", "achieved": head["pass2_gbs"], "peak": peak_gbs, "unit": "GB/s",
                     "frac": head["pass2_gbs"] / peak_gbs, "traffic": tr,
                     "kernel": head["dominant"]["kernel"], "kernel_ms": head["dominant"]["ms"],
                     "algorithmic_bytes_per_launch": head["dominant"]["alg_bytes"] // max(1, head["dominant"]["launches"]),
                     "share_of_step": head["kernels"]["dominant_share_of_step"], "peak_source": peak_src},
        "step_roofline": {"bytes": head["in_bytes"] + head["out_bytes"], "achieved": head["step_gbs"],
                          "peak": peak_gbs, "frac": head["step_gbs"] / peak_gbs,
                          "frac_vs_nominal_8tbs": head["step_gbs"] / 8000.0,
                          "target_ms_60pct_of_8tbs": (head["in_bytes"] + head["out_bytes"]) / (TARGET_FRAC_8TBS * 8000e9) * 1e3,
                          "target_met": head["step_gbs"] / 8000.0 >= TARGET_FRAC_8TBS,
                          "note": "compulsory bytes (one read of the image + one write of every output) / step time"},
        "single_destination": single_line,
        "kernels": head["kernels"],
        "cpu_baseline": cpu,
        "e2e": {k: head["e2e"][k] for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step", "ms_per_step",
                                             "pipeline")},
        "gpu_launches": head["launches_per_step"] * args.steps,
        "clocks": head["clocks"],
        "configs": extra,
        "fhtshift_standalone": shift_lines,
        "angle_range_pruned": pruned_line,
        "peaks": peaks_line,
        "back_to_back": b2b_line,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
