"""World-size-2 gloo test of the multi-GPU host logic: image shards are disjoint
and cover the job, and the step time reported is the max over ranks. CPU only."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1811_06378_b200.sharding import max_over_ranks, rank_images
    imgs = list(rank_images(per_rank, rank, world))
    t = max_over_ranks(10.0 + rank)             # rank-dependent "step time"
    dist.barrier()
    q.put((rank, imgs, t))
    dist.destroy_process_group()


@pytest.mark.parametrize("per_rank", [1, 16])
def test_two_rank_shards_and_max(per_rank):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    owned = sorted(i for _, imgs, _ in res for i in imgs)
    assert owned == list(range(world * per_rank))              # disjoint and complete
    assert all(t == 10.0 + (world - 1) for _, _, t in res)     # every rank sees the max


def test_rank_images_rejects():
    from paper_1811_06378_b200.sharding import rank_images
    with pytest.raises(ValueError):
        rank_images(4, 2, 2)
    with pytest.raises(ValueError):
        rank_images(0, 0, 1)


# ------------------------------------------------------------------ one image over several ranks
def _shard_worker(rank, world, port, P, m, q):
    """Rank `rank` of a sharded full transform, with the oracle standing in for the two passes: pass 1 =
    the first m levels of the Fig. 6 iteration on this rank's strips, laid out in the documented send
    layout [h][z = quadrant][j_local][strip_local][x]; the product's exchange (one all_to_all over gloo);
    pass 2 = the remaining levels on this rank's groups, every other group's rows NaN, so the rows this
    rank keeps can only have come from its own groups."""
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import fht_oracle as O
    from paper_1811_06378_b200.sharding import chunk_offsets, exchange
    from synth import random_image
    img = random_image((P, P), "i32", seed=P).astype(np.float64)
    Hp = P
    K = Hp.bit_length() - 1
    L = K - m
    S, J = (1 << L) // world, (1 << m) // world
    W = 2 * P
    send = np.zeros((world, 4, J, S, W))
    for qd in range(4):
        fr = O.quadrant_frame(img, qd, square_to=(P, P))
        Fm = O.recursion_levels(fr.rows.reshape(Hp, 1, W).copy(), fr.sigma, m)   # [2^L strips][2^m shifts][W]
        for h in range(world):
            for jl in range(J):
                for il in range(S):
                    send[h, qd, jl, il] = Fm[rank * S + il, h * J + jl]
    chunk = 4 * J * S * W * 8
    assert chunk_offsets(chunk, world) == [h * chunk for h in range(world)]
    recv_t = torch.zeros(world * 4 * J * S * W, dtype=torch.float64)
    exchange(torch.from_numpy(send.reshape(-1)), recv_t, world)
    recv = recv_t.numpy().reshape(world, 4, J, S, W)
    ok = True
    for qd in range(4):
        fr = O.quadrant_frame(img, qd, square_to=(P, P))
        Fm = np.full((1 << L, 1 << m, W), np.nan)
        for g in range(world):
            for jl in range(J):
                for il in range(S):
                    Fm[g * S + il, rank * J + jl] = recv[g, qd, jl, il]
        band = O.recursion_levels(Fm, fr.sigma, L)[0][rank * Hp // world:(rank + 1) * Hp // world]
        want = O.hough_of_frame_recursive(fr)[rank * Hp // world:(rank + 1) * Hp // world]
        ok = ok and np.isfinite(band).all() and np.array_equal(band, want)
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,P,m", [(2, 32, 3), (2, 64, 3), (4, 64, 3), (2, 16, 2)])
def test_single_image_shard_exchange(world, P, m):
    """The sharded transform's data flow (fht_shard_pass1 -> one all-to-all -> fht_shard_pass2) on CPU
    ranks with gloo: every rank's band equals the oracle's rows of the whole transform."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, P, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res[r] for r in range(world)), res


def test_chunk_offsets_rejects():
    from paper_1811_06378_b200.sharding import chunk_offsets
    with pytest.raises(ValueError):
        chunk_offsets(16, 0)
