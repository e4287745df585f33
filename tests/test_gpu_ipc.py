"""Two processes on one GPU exchange their per-segment partials through CUDA IPC
mappings of each other's exchange buffers (the multi-process form of the
NVLink one-shot exchange)."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import numpy as np
        import oracle as O
        import paper_2102_01386_b200 as af
        from afinputs import f32_to_bf16_bits, uniform_layout
        # ragged layout: the two shards have different tile counts
        lay = uniform_layout(1_000_003, 7, pre=123_457, head=777)
        fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="bf16", rank=rank, world=world)
        assert fm.set_peers_ipc()
        oz = O.Freezer(lay.offsets, lay.kinds, O.DT_BF16)
        scale = np.random.default_rng(5).random(lay.n_segments) * 0.5 + 0.3
        out = []
        for T in range(5):
            for t in range(2):
                rng = np.random.default_rng([5, T, t])
                x = rng.standard_normal(lay.n).astype(np.float32)
                x *= np.repeat((scale ** T).astype(np.float32), np.diff(lay.offsets)) * np.float32(1e-3)
                g = f32_to_bf16_bits(x)
                gd = torch.from_numpy(g.view(np.int16)).view(torch.bfloat16).cuda()
                if t == 1:
                    fm.interval_end(gd)
                else:
                    fm.layer_norms(gd)
                oz.layer_norms(g, t == 1)
            d = fm.decision()
            o = oz.update_and_decide()
            assert not d["flags"] & 32, "exchange timeout"
            if not (d["flags"] | o["flags"]) & 4:
                assert d["boundary_after"] == o["boundary_after"]
            np.testing.assert_allclose(d["norm"], o["norm"], rtol=1e-12)
            out.append((d["boundary_after"], d["norm"]))
        allr = [None] * world
        dist.all_gather_object(allr, out)
        assert allr[0] == allr[1]
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.timeout(600)
def test_two_processes_ipc_exchange_one_gpu():
    assert torch.cuda.is_available()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=500) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def _rs_worker(rank, world, port, q):
    """NEXT 1 (ZeRO form) across processes: every rank maps every rank's gradient
    buffer and the barrier flags through CUDA IPC; the two processes time-share
    the one GPU, so each barrier is crossed when the other process's kernel runs."""
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import numpy as np
        import oracle as O
        import paper_2102_01386_b200 as af
        from afinputs import f32_to_bf16_bits, uniform_layout
        lay = uniform_layout(500_009, 6, pre=40_001, head=333)
        fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="bf16", rank=rank, world=world)
        assert fm.set_peers_ipc()
        grad = torch.zeros(lay.n, dtype=torch.bfloat16, device="cuda")
        fm.set_grad_peers_ipc(grad)
        fm.set_grad_peers_ipc(grad)    # re-registration maps each peer allocation once (shared mapping)
        fm.set_max_ctas(32)
        info = fm.info()
        sb, se = info["shard_begin"], info["shard_end"]
        out = torch.zeros(se - sb, device="cuda")
        oz = O.Freezer(lay.offsets, lay.kinds, O.DT_F32)
        scale = np.random.default_rng(9).random(lay.n_segments) * 0.5 + 0.3
        res = []
        for T in range(4):
            for t in range(2):
                gs_in = []
                for r in range(world):
                    rng = np.random.default_rng([9, T, t, r])
                    x = rng.standard_normal(lay.n).astype(np.float32)
                    x *= np.repeat((scale ** T).astype(np.float32), np.diff(lay.offsets)) * np.float32(1e-3)
                    gs_in.append(f32_to_bf16_bits(x))
                grad.copy_(torch.from_numpy(gs_in[rank].view(np.int16)).view(torch.bfloat16).cuda())
                f_before = oz.f
                fm.reduce_scatter_step(out, interval_end=(t == 1))
                torch.cuda.synchronize()
                gs = O.reduce_gradients(gs_in, O.DT_BF16, 1.0 / world)
                oh = out.cpu().numpy()
                for l in O.active_segments(lay.kinds, f_before):
                    lo, hi = max(lay.offsets[l], sb), min(lay.offsets[l + 1], se)
                    if lo < hi:
                        assert np.array_equal(oh[lo - sb:hi - sb], gs[lo:hi])
                oz.layer_norms(gs, t == 1)
            d = fm.decision()
            o = oz.update_and_decide()
            assert not d["flags"] & 32, "barrier timeout"
            if not (d["flags"] | o["flags"]) & 4:
                assert d["boundary_after"] == o["boundary_after"]
            np.testing.assert_allclose(d["norm"], o["norm"], rtol=1e-12)
            res.append((d["boundary_after"], d["norm"]))
        allr = [None] * world
        dist.all_gather_object(allr, res)
        assert allr[0] == allr[1]
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.timeout(600)
def test_two_processes_fused_reduce_scatter_one_gpu():
    assert torch.cuda.is_available()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rs_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=500) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
