"""World-size-2 CPU tests (gloo) of the multi-rank host logic: NCCL-id
bootstrap through torch.distributed, the library's contiguous shard bounds,
rank-order combination of per-segment partials and replicated decisions.
The per-shard arithmetic here is the oracle's (test infrastructure); the GPU
sharded path is covered by the fake-P parity test and by torchrun on B200s."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, active=False):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        import paper_2102_01386_b200 as af
        from afinputs import bert_grad_step, uniform_layout
        # 1) NCCL unique id bootstrap: identical 128 bytes on every rank
        uid = af.bootstrap_nccl_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert len(uid) == 128 and all(u == ids[0] for u in ids) and any(uid)
        # 2) shard bounds from the library (host-only create)
        lay = uniform_layout(1_000_003, 7, pre=123_457, head=777)
        fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="bf16", rank=rank, world=world, bind=False,
                               shard_active=active)
        info = fm.info()
        sb, se = info["shard_begin"], info["shard_end"]
        bounds = [None] * world
        dist.all_gather_object(bounds, (sb, se))
        assert bounds[0][0] == 0 and bounds[-1][1] == lay.n
        assert all(bounds[r][1] == bounds[r + 1][0] for r in range(world - 1))
        # 3) per-rank partial sums over the shard, all-gathered, summed in rank order
        full = O.Freezer(lay.offsets, lay.kinds, O.DT_BF16)
        local = O.Freezer(lay.offsets, lay.kinds, O.DT_BF16)
        decisions = []
        for T in range(6):
            # active-suffix shards: this interval's shard is the library's split of the
            # active suffix for the current boundary (static: the same every interval)
            sb, se = fm.shard_of(full.f)
            bnd = [None] * world
            dist.all_gather_object(bnd, (sb, se))
            assert all(bnd[r][1] == bnd[r + 1][0] for r in range(world - 1)) and bnd[-1][1] == lay.n
            for t in range(2):
                g = bert_grad_step(lay, 3, T, t, dtype="bf16")
                gl = g.copy()
                gl[:sb] = 0
                gl[se:] = 0                    # the rank only reads its shard
                full.layer_norms(g, t == 1)
                local.layer_norms(gl, t == 1)
            rows = torch.from_numpy(local.pending.copy())
            gathered = [torch.zeros_like(rows) for _ in range(world)]
            dist.all_gather(gathered, rows)
            ss = np.zeros(lay.n_segments)
            for r in range(world):                # rank order 0..P-1
                ss = ss + gathered[r].numpy()
            np.testing.assert_allclose(ss, full.pending, rtol=1e-13)
            local.pending = ss
            rec_local = local.update_and_decide()
            rec_full = full.update_and_decide()
            assert rec_local["boundary_after"] == rec_full["boundary_after"]
            thr = rec_local["threshold"]
            decisions.append((rec_local["boundary_after"], None if thr != thr else thr))
        allr = [None] * world
        dist.all_gather_object(allr, decisions)
        assert all(a == allr[0] for a in allr)        # replicated, identical decisions
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("active", [False, True])
def test_two_rank_gloo_host_logic(active):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q, active)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
