"""Multi-GPU host logic. Two ways the path shards:

* Independent images (weak scaling, the bench's --gpus N): rank r of N transforms the global images
  [r*B, (r+1)*B); the only collective is the max over ranks of the measured step time.
* One image over N GPUs (`full_sharded`): pass 1 on each rank's strips, ONE all-to-all of
  the pass-1 scratch, pass 2 on each rank's groups; rank h ends with output rows [h Hp/N, (h+1) Hp/N) of
  every quadrant (fht_shard_* in include/fht.h). The exchange either goes through NCCL
  (torch.distributed.all_to_all_single on the send buffer pass 1 filled) or, with `recv_peers` (the
  receive buffers of every rank mapped into this process: peer memory over NVLink / NVSwitch), happens
  in pass 1's own stores -- then one barrier replaces the collective.

Pure plumbing: argument marshalling and torch.distributed calls; every step of the transform runs in the
CUDA kernels behind the C ABI.
"""
from __future__ import annotations

import ctypes


def rank_images(per_rank: int, rank: int, world: int) -> range:
    """Global image indices owned by `rank` (weak scaling: every rank owns `per_rank` images)."""
    if per_rank < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard request")
    return range(rank * per_rank, (rank + 1) * per_rank)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over the default process group (identity when not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def chunk_offsets(chunk_bytes: int, world: int) -> list[int]:
    """Byte offset of rank h's chunk in a send buffer (and of rank g's chunk in a receive buffer):
    the all-to-all moves equal chunks, chunk h of every rank's send buffer to rank h."""
    if chunk_bytes < 0 or world < 1:
        raise ValueError("bad chunk layout")
    return [h * chunk_bytes for h in range(world)]


def exchange(send, recv, world: int, group=None) -> None:
    """The one collective of a sharded transform: chunk h of `send` on every rank lands as chunk
    (sender) of `recv` on rank h. torch.distributed with NCCL on GPUs (gloo in the CPU tests)."""
    import torch.distributed as dist
    if world == 1:
        recv.copy_(send)
        return
    dist.all_to_all_single(recv, send, group=group)


def shard_describe(t, world: int, rank: int):
    """fht_shard_describe for the image tensor t ([h][w] or [B][h][w], on the device)."""
    from . import _image, _lib
    img, _ = _image(t)
    sh = _lib.FhtShard()
    _lib.check("fht_shard_describe", _lib.lib.fht_shard_describe(ctypes.byref(img), int(world), int(rank),
                                                                 ctypes.byref(sh)))
    return sh


def shard_pass1(t, sh, dst_ptrs) -> int:
    """Pass 1 of rank sh.rank: dst_ptrs[h] = device address where rank h's chunk goes."""
    import torch
    from . import _image, _lib
    img, t = _image(t)
    arr = (ctypes.c_void_p * sh.world)(*[ctypes.c_void_p(int(p)) for p in dst_ptrs])
    st = ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)
    return _lib.check("fht_shard_pass1", _lib.lib.fht_shard_pass1(ctypes.byref(img), ctypes.byref(sh), arr, st))


def shard_pass2(t, sh, recv, shifted: bool = False, pair: bool = False):
    """Pass 2 of rank sh.rank from the receive buffer: this rank's band (and / or its fhtshift)."""
    import torch
    from . import HoughImage, _DT_OUT, _image, _lib
    img, t = _image(t)
    res = []
    for want in (pair or not shifted, pair or shifted):
        if not want:
            res.append(None)
            continue
        d = _lib.FhtHough.from_buffer_copy(sh.band)
        storage = torch.empty(d.batch * d.batch_stride, dtype=_DT_OUT[d.dtype], device=t.device)
        d.data = storage.data_ptr()
        res.append(HoughImage(storage, d))
    st = ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)
    n = _lib.check("fht_shard_pass2", _lib.lib.fht_shard_pass2(
        ctypes.byref(img), ctypes.byref(sh), ctypes.c_void_p(recv.data_ptr()),
        ctypes.byref(res[0].desc) if res[0] is not None else None,
        ctypes.byref(res[1].desc) if res[1] is not None else None, st))
    for h in res:
        if h is not None:
            h.launches = n
    if pair:
        return res[0], res[1]
    return res[1] if shifted else res[0]


def full_sharded(t, group=None, shifted: bool = False, pair: bool = False, recv_peers=None, recv=None):
    """Full four-quadrant transform of t sharded over the ranks of `group` (default: the default process
    group; one process = world 1). Every rank passes the same image; rank h returns the band of output rows
    [h Hp/N, (h+1) Hp/N) of every quadrant (`.desc.row0` = its first row).

    recv_peers: optional list of N device addresses, the receive buffers of ranks 0..N-1 mapped into this
    process (each `sh.recv_bytes`); this rank's own must be `recv`. Pass 1 then writes every chunk
    straight into its owner's buffer and a barrier stands in for the all-to-all."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    sh = shard_describe(t, world, rank)
    if recv is None:
        recv = torch.empty(sh.recv_bytes, dtype=torch.uint8, device=t.device)
    offs = chunk_offsets(sh.chunk_bytes, world)
    if recv_peers is not None:
        if len(recv_peers) != world:
            raise ValueError("recv_peers needs one address per rank")
        shard_pass1(t, sh, [int(recv_peers[h]) + offs[rank] for h in range(world)])
        torch.cuda.current_stream(t.device).synchronize()
        if world > 1:
            dist.barrier(group=group)        # every rank's chunks have landed in every receive buffer
    else:
        send = torch.empty(sh.send_bytes, dtype=torch.uint8, device=t.device)
        shard_pass1(t, sh, [send.data_ptr() + o for o in offs])
        exchange(send, recv, world, group)
    return shard_pass2(t, sh, recv, shifted=shifted, pair=pair)
