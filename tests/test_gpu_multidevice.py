"""Multi-GPU paths across real devices: one process per
GPU, ranks on DIFFERENT devices, so the exchange and the fused reduce-scatter
cross NVLink.  Runs whenever >= 2 CUDA devices are visible (skipped on the
one-GPU boxes of this build; the same flows run two-ranks-on-one-GPU in
test_gpu_ipc.py / test_gpu_parity.py):

  * the in-kernel NVLink one-shot exchange over CUDA IPC peer mappings;
  * the NCCL fallback (all-gather of the per-layer partials + decide kernel);
  * the fused reduce-scatter + accumulate (NEXT 1, ZeRO form) at P = 2;
  * single-process contexts on two devices with local peers (peer access
    enabled by the library) and the cross-GPU cache get (NEXT 4).

Decisions are compared with the fp64 oracle on the same seeded inputs and must
be identical on every rank."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs >= 2 CUDA devices")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grad(lay, seed, T, t, r=0):
    import numpy as np
    from afinputs import f32_to_bf16_bits
    scale = np.random.default_rng(seed).random(lay.n_segments) * 0.5 + 0.3
    rng = np.random.default_rng([seed, T, t, r])
    x = rng.standard_normal(lay.n).astype(np.float32)
    x *= np.repeat((scale ** T).astype(np.float32), np.diff(lay.offsets)) * np.float32(1e-3)
    return f32_to_bf16_bits(x)


def _worker(rank, world, port, mode, q):
    try:
        import numpy as np
        import torch.distributed as dist

        import oracle as O
        import paper_2102_01386_b200 as af
        from afinputs import uniform_layout
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(rank)
        lay = uniform_layout(2_000_003, 9, pre=200_001, head=777)
        fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="bf16", rank=rank, world=world)
        if mode == "p2p":
            assert fm.set_peers_ipc(), "CUDA IPC peer mappings across devices failed"
        elif mode == "nccl":
            fm.set_comm()
        out = []
        if mode in ("p2p", "nccl"):
            oz = O.Freezer(lay.offsets, lay.kinds, O.DT_BF16)
            for T in range(5):
                for t in range(2):
                    g = _grad(lay, 5, T, t)
                    gd = torch.from_numpy(g.view(np.int16)).view(torch.bfloat16).cuda()
                    if t == 1:
                        fm.interval_end(gd)
                    else:
                        fm.layer_norms(gd)
                    oz.layer_norms(g, t == 1)
                d, o = fm.decision(), oz.update_and_decide()
                assert not d["flags"] & 32, "exchange timeout"
                if not (d["flags"] | o["flags"]) & 4:
                    assert d["boundary_after"] == o["boundary_after"], (T, d["boundary_after"], o["boundary_after"])
                np.testing.assert_allclose(d["norm"], o["norm"], rtol=1e-12)
                out.append((d["boundary_after"], d["norm"]))
        else:  # fused reduce-scatter across devices
            assert fm.set_peers_ipc()
            grad = torch.zeros(lay.n, dtype=torch.bfloat16, device="cuda")
            fm.set_grad_peers_ipc(grad)
            info = fm.info()
            sb, se = info["shard_begin"], info["shard_end"]
            rs_out = torch.zeros(se - sb, device="cuda")
            oz = O.Freezer(lay.offsets, lay.kinds, O.DT_F32)
            for T in range(4):
                for t in range(2):
                    gs_in = [_grad(lay, 9, T, t, r) for r in range(world)]
                    grad.copy_(torch.from_numpy(gs_in[rank].view(np.int16)).view(torch.bfloat16).cuda())
                    dist.barrier()
                    f_before = oz.f
                    fm.reduce_scatter_step(rs_out, interval_end=(t == 1))
                    torch.cuda.synchronize()
                    gs = O.reduce_gradients(gs_in, O.DT_BF16, 1.0 / world)
                    oh = rs_out.cpu().numpy()
                    for l in O.active_segments(lay.kinds, f_before):
                        lo, hi = max(lay.offsets[l], sb), min(lay.offsets[l + 1], se)
                        if lo < hi:
                            assert np.array_equal(oh[lo - sb:hi - sb], gs[lo:hi])
                    oz.layer_norms(gs, t == 1)
                    dist.barrier()
                d, o = fm.decision(), oz.update_and_decide()
                assert not d["flags"] & 32, "barrier timeout"
                if not (d["flags"] | o["flags"]) & 4:
                    assert d["boundary_after"] == o["boundary_after"]
                np.testing.assert_allclose(d["norm"], o["norm"], rtol=1e-12)
                out.append((d["boundary_after"], d["norm"]))
        allr = [None] * world
        dist.all_gather_object(allr, out)
        assert allr[0] == allr[1], "ranks took different decisions"
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.timeout(900)
@pytest.mark.parametrize("mode", ["p2p", "nccl", "reduce_scatter"])
def test_two_devices_two_processes(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=800) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


@pytest.mark.timeout(600)
def test_one_process_two_devices_local_peers_and_global_cache():
    """Contexts bound on cuda:0 and cuda:1 in one process: set_peers_local enables
    peer access and the interval ends exchange over NVLink; a rank's cache get of
    the other rank's ids reads its store through peer memory."""
    import threading

    import numpy as np

    import oracle as O
    import paper_2102_01386_b200 as af
    from afinputs import cache_rows, uniform_layout
    lay = uniform_layout(1_000_003, 7, pre=123_457, head=777)
    fms = []
    for r in range(2):
        with torch.cuda.device(r):
            fms.append(af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="bf16", rank=r, world=2,
                                         device=torch.device("cuda", r)))
    for r in range(2):
        with torch.cuda.device(r):
            fms[r].set_peers_local(fms)
    oz = O.Freezer(lay.offsets, lay.kinds, O.DT_BF16)
    for T in range(4):
        for t in range(2):
            g = _grad(lay, 13, T, t)
            # both ranks' kernels must run concurrently (each waits for the other's row)
            def run(r):
                with torch.cuda.device(r):
                    gd = torch.from_numpy(g.view(np.int16)).view(torch.bfloat16).to(f"cuda:{r}")
                    (fms[r].interval_end if t == 1 else fms[r].layer_norms)(gd)
                    torch.cuda.synchronize(r)
            th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
            for x in th:
                x.start()
            for x in th:
                x.join()
            oz.layer_norms(g, t == 1)
        o = oz.update_and_decide()
        d = [fms[r].decision() for r in range(2)]
        assert d[0]["boundary_after"] == d[1]["boundary_after"]
        np.testing.assert_allclose(d[0]["norm"], o["norm"], rtol=1e-12)
    # cross-GPU cache get (NEXT 4)
    num, rb = 1000, 4096 + 16
    caches = []
    for r in range(2):
        with torch.cuda.device(r):
            caches.append(af.ActivationCache(num, rb, rank=r, world=2, device=torch.device("cuda", r)))
    for r in range(2):
        with torch.cuda.device(r):
            caches[r].set_peers_local(caches)
    ids = np.arange(0, 200, 2) + 1          # rank 1's ids
    rows = cache_rows(1, 1, len(ids), rb)
    with torch.cuda.device(1):
        caches[1].put(torch.from_numpy(ids).to("cuda:1"), torch.from_numpy(rows).to("cuda:1"), 3)
        torch.cuda.synchronize(1)
    with torch.cuda.device(0):
        out = torch.zeros((len(ids), rb), dtype=torch.uint8, device="cuda:0")
        dep = torch.zeros(len(ids), dtype=torch.int32, device="cuda:0")
        caches[0].get_global(torch.from_numpy(ids).to("cuda:0"), 3, out, dep)
        torch.cuda.synchronize(0)
        assert np.array_equal(out.cpu().numpy(), rows) and set(dep.cpu().tolist()) == {3}
