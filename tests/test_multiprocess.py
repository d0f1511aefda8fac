"""The N>1 path on CPU: world_size 2 over gloo.  Each rank traces its weak
shard of rays (oracle as the per-ray engine stand-in on CPU), builds the K7
histogram, and the all-reduced histogram must equal the single-process one --
the same host logic bench.py runs over NCCL on GPUs."""
import os
import socket

import numpy as np
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


def _rank_main(rank, world, port, paths, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_2112_05570_b200.sharding import allreduce_histogram, histogram_host, weak_shard
    sh = weak_shard(rank, world, N_PER_RANK)
    m = orc.Mesh.from_files(*paths)
    r = orc.raygen(0, (0.0, 0.0, 1.0, 1.0), 0, sh.first, sh.count)
    o = m.trace(r)
    h = torch.from_numpy(histogram_host(o["seg"], o["steps"], o["status"]))
    allreduce_histogram(h)
    if rank == 0:
        np.save(out_path, h.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_histogram_allreduce(tmp_path):
    from oracle import oracle as orc
    from paper_2112_05570_b200.sharding import histogram_host
    paths = fixture_paths("lines1024", "cdt")
    out = str(tmp_path / "h.npy")
    mp.start_processes(_rank_main, args=(2, _free_port(), paths, out), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    m = orc.Mesh.from_files(*paths)
    o = m.trace(orc.raygen(0, (0.0, 0.0, 1.0, 1.0), 0, 0, 2 * N_PER_RANK))
    ref = histogram_host(o["seg"], o["steps"], o["status"])
    assert np.array_equal(got, ref)
    assert got[:1024].sum() == 2 * N_PER_RANK
