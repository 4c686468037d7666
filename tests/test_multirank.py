"""World-size-2 (gloo, CPU) coverage of the multi-rank path: disjoint shards
of the seeded stream, no data exchange, max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0710_0510_b200.sharding import max_over_ranks, shard, weak_shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_per_rank, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    first, count = weak_shard(rank, n_per_rank)
    dr = O.draws(0x07100512, count * 7, 128, start=first * 7).reshape(count, 7).astype(np.uint64)
    w = np.zeros(count, np.uint64)
    for j in range(7):
        w = w * np.uint64(128) + dr[:, j]
    res = O.redq_f64(5, 128, 6, w.astype(np.float64), float_mode=True, window=4)
    np.save(os.path.join(outdir, f"r{rank}.npy"), res)
    m = max_over_ranks(float(rank + 1) * 1.5, dist, "cpu")
    np.save(os.path.join(outdir, f"max{rank}.npy"), np.array([m]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_partition():
    for n in (0, 1, 7, 1000, 1 << 26):
        for world in (1, 2, 3, 8):
            parts = [shard(r, world, n) for r in range(world)]
            assert sum(c for _, c in parts) == n
            assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(world - 1))


def test_two_ranks_gloo(tmp_path, orc):
    world, n = 2, 3000
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n, str(tmp_path)), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(world)])
    # the ranks' shards tile the single-process stream exactly
    dr = orc.draws(0x07100512, world * n * 7, 128).reshape(world * n, 7).astype(np.uint64)
    w = np.zeros(world * n, np.uint64)
    for j in range(7):
        w = w * np.uint64(128) + dr[:, j]
    assert (got == orc.redq_f64(5, 128, 6, w.astype(np.float64), float_mode=True, window=4)).all()
    assert all(float(np.load(tmp_path / f"max{r}.npy")[0]) == 3.0 for r in range(world))


@pytest.mark.gpu
def test_rank_shards_on_the_device_tile_the_stream(qpk, orc, torch_cuda):
    """The per-rank work of bench.py's multi-GPU path on the product itself:
    each rank of a world of 4 generates its shard of the seeded C2 stream on
    the device (gen_words at the rank's first word) and reduces it with the
    library's REDQ kernel; concatenated, the shards equal the single-process
    stream's residues (the ranks run one after another on this GPU: they
    never wait on one another, and the only collectives of the real run are
    the timing barrier and the max-over-ranks of the elapsed time)."""
    torch = torch_cuda
    world, n = 4, 70001
    plan = qpk.RedqPlan(5, 128, 6, qpk.FLOAT_PREMUL).attach_correction(4)
    parts = []
    for rank in range(world):
        first, count = weak_shard(rank, n)
        w = torch.empty(count, dtype=torch.float64, device="cuda")
        qpk.gen_words(qpk.C2.seed, count, 128, 6, w, first=first)
        parts.append(plan.residues(w).cpu().numpy())
    plan.sync()
    got = np.concatenate(parts)
    dr = orc.draws(qpk.C2.seed, world * n * 7, 128).reshape(world * n, 7).astype(np.uint64)
    w = np.zeros(world * n, np.uint64)
    for j in range(7):
        w = w * np.uint64(128) + dr[:, j]
    assert (got == orc.redq_f64(5, 128, 6, w.astype(np.float64), float_mode=True, window=4)).all()
