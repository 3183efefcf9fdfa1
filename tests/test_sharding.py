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
