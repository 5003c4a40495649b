"""Multi-process (world_size 2, gloo, CPU) coverage of the frame-sharded
multi-GPU layer, driving the product's protocol: frame assignment
(frames_for_rank), the frame export format (sharding.export_*), the
point-to-point FrameGather transport and merge_sharded's in-order merge on
rank 0, and the max/sum timer reductions. Per-frame results come from the
CPU oracle on tiny frames (no GPU here); on a GPU box the same protocol
carries FrameOutput.export payloads over NCCL (pipeline.run_sequence_sharded)."""

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


CFG = dict(stage_lo=(-1000, -1000, 0), stage_hi=(1000, 1000, 1000), coarse_spacing=80.0,
           fine_spacing=40.0, t_small=3)


def _frame(sils, f):
    return [np.roll(m, 7 * f, axis=1) for m in sils]  # a different frame per index


def _oracle_frame(rig, sils, f):
    import oracle as O

    c = CFG
    return O.run_frame(rig, _frame(sils, f), c["stage_lo"], c["stage_hi"], c["coarse_spacing"],
                       c["fine_spacing"], 1, c["t_small"])


def _export(out):
    from paper_1903_11785_b200.sharding import export_from_arrays

    v, t, _ = out["merged"]
    cids = [int(cid) for _, _, cid in out["rois"]]
    info, vb, tb = [], 0, 0
    for mv, mt, _ in out["meshes"]:
        info.append([vb, len(mv), 0, 0, tb, len(mt), 0, 0])
        vb, tb = vb + len(mv), tb + len(mt)
    vis = out["visibility"]
    stride = max((len(t) + 31) // 32, 1)
    bits = np.zeros((len(vis), stride), dtype=np.uint32)
    for row, cid in enumerate(sorted(vis)):
        packed = np.packbits(np.r_[vis[cid], np.zeros(32 * stride - len(t), bool)],
                             bitorder="little")
        bits[row] = packed.view(np.uint32)
    ms = [0.5, 0.25, 1.0, 2.0, 3.0, 0.125]
    return export_from_arrays(out["stats"], ms, cids, np.array(info).reshape(-1, 8), v, t, bits)


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    import golden_io as G
    from paper_1903_11785_b200 import sharding
    from paper_1903_11785_b200.pipeline import PipelineConfig

    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_frames = 5
    z = G.load("tiny_cli")
    rig, sils = G.rig(z), G.sils(z)
    cfg = PipelineConfig(**CFG)
    mine = sharding.frames_for_rank(rank, world, n_frames)

    def local():  # this rank's frames, in assignment order, as the GPU lanes yield them
        for f in mine:
            meta, payload = _export(_oracle_frame(rig, sils, f))
            bundle = sharding.bundle_from_export(meta, payload, cfg, rig, f) if rank == 0 else None
            yield f, bundle, None, (meta, payload, None)

    gather = sharding.frame_gather()
    got = list(sharding.merge_sharded(
        rank, world, n_frames, local(), gather,
        lambda f, meta, payload, ev: sharding.bundle_from_export(meta, payload, cfg, rig, f)))
    t_max = sharding.reduce_max(float(rank + 1))
    t_sum = sharding.reduce_sum(float(len(mine)))
    if rank == 0:
        ok = [f == i for i, (f, _, _) in enumerate(got)]
        for f, bundle, _ in got:  # every frame, whichever rank computed it, equals the oracle
            ref = _oracle_frame(rig, sils, f)
            m = bundle.merged_mesh
            ok.append(bundle.frame_id == f)
            ok.append(bundle.stats == {k: int(v) for k, v in ref["stats"].items()})
            ok.append(np.array_equal(m.vertices, ref["merged"][0]))
            ok.append(np.array_equal(m.triangles, ref["merged"][1]))
            ok.append(np.array_equal(m.object_ids, ref["merged"][2]))
            ok.append(all(np.array_equal(bundle.visibility[c], ref["visibility"][c])
                          for c in ref["visibility"]))
            ok.append(len(bundle.meshes) == len(ref["meshes"]) and all(
                np.array_equal(a.triangles, b[1]) for a, b in zip(bundle.meshes, ref["meshes"])))
        np.save(os.path.join(out_dir, "summary.npy"),
                np.array([t_max, t_sum, len(got), float(all(ok))], dtype=np.float64))
    else:
        np.save(os.path.join(out_dir, f"rank{rank}.npy"),
                np.array([f for f, b, _ in got if b is None], dtype=np.float64))
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
    t_max, t_sum, n, ok = np.load(tmp_path / "summary.npy")
    assert t_max == 2.0  # slowest rank wins
    assert t_sum == 5.0  # every frame assigned exactly once
    assert int(n) == 5 and ok == 1.0  # rank 0 holds all 5 frames, in order, oracle-equal
    assert list(np.load(tmp_path / "rank1.npy")) == [1.0, 3.0]  # rank 1 sent its frames
