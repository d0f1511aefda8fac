"""The N>1 path on CPU: world_size 2 over gloo.  Each rank traces its shard
of rays (strong: the bench default, 2 * N_PER_RANK split; weak: N_PER_RANK
each) in the bench's coherent generator order (oracle as the per-ray engine
stand-in on CPU), builds the K7 histogram, and the all-reduced histogram must
equal the single-process one; the bench's max-over-ranks timing reduction is
checked too -- the same host logic bench.py runs over NCCL on GPUs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import fixture_paths

N_PER_RANK = 3000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, paths, out_path, scaling):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import oracle as orc
    from paper_2112_05570_b200.sharding import (allreduce_histogram, histogram_host, max_over_ranks,
                                                strong_shard, weak_shard)
    sh = strong_shard(rank, world, 2 * N_PER_RANK) if scaling == "strong" else weak_shard(rank, world, N_PER_RANK)
    m = orc.Mesh.from_files(*paths)
    r = orc.raygen(bench.mode_word(0, "coherent"), (0.0, 0.0, 1.0, 1.0), 0, sh.first, sh.count)
    o = m.trace(r)
    h = torch.from_numpy(histogram_host(o["seg"], o["steps"], o["status"]))
    allreduce_histogram(h)
    worst = max_over_ranks(float(rank) + 0.5)
    if rank == 0:
        np.save(out_path, h.numpy())
        np.save(out_path + ".max.npy", np.array([worst]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_two_rank_histogram_allreduce(tmp_path, scaling):
    import bench
    from oracle import oracle as orc
    from paper_2112_05570_b200.sharding import histogram_host
    paths = fixture_paths("lines1024", "cdt")
    out = str(tmp_path / "h.npy")
    mp.start_processes(_rank_main, args=(2, _free_port(), paths, out, scaling), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    m = orc.Mesh.from_files(*paths)
    o = m.trace(orc.raygen(bench.mode_word(0, "coherent"), (0.0, 0.0, 1.0, 1.0), 0, 0, 2 * N_PER_RANK))
    ref = histogram_host(o["seg"], o["steps"], o["status"])
    assert np.array_equal(got, ref)
    assert got[:1024].sum() == 2 * N_PER_RANK
    assert float(np.load(out + ".max.npy")[0]) == 1.5  # max over ranks of rank + 0.5


def test_shards_cover_the_ray_range():
    from paper_2112_05570_b200.sharding import strong_shard, weak_shard
    for world in (1, 2, 3, 8):
        for total in (0, 1, 7, 1 << 26):
            sh = [strong_shard(r, world, total) for r in range(world)]
            assert sh[0].first == 0 and sum(x.count for x in sh) == total
            assert all(a.first + a.count == b.first for a, b in zip(sh, sh[1:]))
            assert max(x.count for x in sh) - min(x.count for x in sh) <= 1
        w = [weak_shard(r, world, 5) for r in range(world)]
        assert [x.first for x in w] == [5 * r for r in range(world)]
    with pytest.raises(ValueError):
        strong_shard(2, 2, 10)
