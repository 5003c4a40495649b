"""Multi-process (world_size 2, gloo, CPU) coverage of the frame-sharded
multi-GPU layer: disjoint complete frame assignment, max/sum timer
reductions, and gathering per-frame results (computed here by the CPU
oracle on two tiny frames) to rank 0 in frame order."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    import golden_io as G
    import oracle as O
    from paper_1903_11785_b200 import sharding

    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_frames = 5
    mine = sharding.frames_for_rank(rank, world, n_frames)
    z = G.load("tiny_cli")
    rig, sils = G.rig(z), G.sils(z)
    results = {}
    for f in mine[:2]:
        s = [np.roll(m, f, axis=1) for m in sils]  # a different frame per index
        out = O.run_frame(rig, s, (-1000, -1000, 0), (1000, 1000, 1000), 80.0, 40.0, 1, 3)
        results[f] = (out["stats"]["triangles"], out["merged"][1][:5].copy())
    t_max = sharding.reduce_max(float(rank + 1))
    t_sum = sharding.reduce_sum(float(len(mine)))
    gathered = sharding.gather_to_rank0(results)
    if rank == 0:
        np.save(os.path.join(out_dir, "summary.npy"),
                np.array([t_max, t_sum, len(gathered)] + list(gathered.keys()), dtype=np.float64))
    dist.destroy_process_group()


def test_frame_assignment_is_a_partition():
    from paper_1903_11785_b200.sharding import frames_for_rank

    for world in (1, 2, 3, 8):
        parts = [frames_for_rank(r, world, 300) for r in range(world)]
        flat = sorted(f for p in parts for f in p)
        assert flat == list(range(300))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        frames_for_rank(2, 2, 10)


def test_two_rank_gloo_sharded_frames(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    summary = np.load(tmp_path / "summary.npy")
    t_max, t_sum, n = summary[:3]
    assert t_max == 2.0  # slowest rank wins
    assert t_sum == 5.0  # every frame assigned exactly once
    assert int(n) == 4 and list(summary[3:]) == [0.0, 1.0, 2.0, 3.0]
