"""Thin Python binding over libautofreeze (include/af.h), same names as the ABI.

PyTorch supplies device memory (workspace, cache storage), streams/events and
torch.distributed for the NCCL-id bootstrap.  Every step of the path runs in the
library's sm_100a kernels; nothing here computes.
"""
import ctypes
import os
from ctypes import byref, c_int64, c_size_t, c_uint32, c_void_p

import torch

from . import _lib as L
from ._lib import check, lib

_DTYPES = {"f32": L.AF_DT_F32, "fp32": L.AF_DT_F32, torch.float32: L.AF_DT_F32,
           "bf16": L.AF_DT_BF16, torch.bfloat16: L.AF_DT_BF16}
_PCT = {"linear": L.AF_PCT_LINEAR, "nearest_rank": L.AF_PCT_NEAREST_RANK}
_ACC = {"delta": L.AF_ACC_DELTA, "step_sumsq": L.AF_ACC_STEP_SUMSQ}


def _stream_handle(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return c_void_p(s.cuda_stream)


def _dev_tensor(t, name, device, min_bytes=0, dtypes=None, min_numel=0):
    """Argument checks at the binding boundary (the C ABI takes raw pointers and
    cannot see sizes): on `device`, contiguous, of an accepted dtype, large enough."""
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.device.type != "cuda" or (device is not None and t.device != torch.device(device)):
        raise ValueError(f"{name} must live on {device} (got {t.device})")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtypes is not None and t.dtype not in dtypes:
        raise TypeError(f"{name} must have dtype in {[str(d) for d in dtypes]} (got {t.dtype})")
    if t.numel() * t.element_size() < min_bytes or t.numel() < min_numel:
        raise ValueError(f"{name} is too small ({t.numel()} elements of {t.element_size()} B)")
    return t


_GRAD_TORCH = {L.AF_DT_F32: (torch.float32,), L.AF_DT_BF16: (torch.bfloat16, torch.int16)}


def decision_to_dict(rec, n_segments):
    return dict(interval=rec.interval, boundary_before=rec.boundary_before,
                boundary_after=rec.boundary_after, n_active=rec.n_active,
                threshold=rec.threshold, flags=rec.flags, near_tie_seg=rec.near_tie_seg,
                sumsq=list(rec.sumsq[:n_segments]), norm=list(rec.norm[:n_segments]),
                eta=list(rec.eta[:n_segments]))


class FreezingModule:
    """af_ctx: the per-GPU Freezing Module (§3.4, Alg. 1).

    offsets: L+1 element offsets of the flat gradient buffer; kinds: L segment
    kinds (0 PRE, 1 POOL, 2 HEAD) in the order PRE* POOL+ HEAD*."""

    def __init__(self, offsets, kinds, grad_dtype="bf16", percentile=50.0, pct_method="linear",
                 acc_mode="delta", tie_rel_eps=1e-5, min_active=2, rank=0, world=1, device=None,
                 bind=True, shard_active=False):
        self.offsets = [int(o) for o in offsets]
        self.kinds = [int(k) for k in kinds]
        self.n_segments = len(self.kinds)
        self._offs = (ctypes.c_int64 * len(self.offsets))(*self.offsets)
        self._kinds = (ctypes.c_int32 * max(1, len(self.kinds)))(*self.kinds)
        lay = L.AfLayout(len(self.kinds), self._offs, self._kinds, _DTYPES[grad_dtype])
        cfg = L.AfConfig(float(percentile), _PCT[pct_method], _ACC[acc_mode], float(tie_rel_eps),
                         int(min_active), int(rank), int(world), 1 if shard_active else 0)
        h = c_void_p()
        check(lib.af_ctx_create(byref(lay), byref(cfg), byref(h)), "af_ctx_create")
        self._h = h
        self.grad_dtype = _DTYPES[grad_dtype]
        self.rank, self.world = int(rank), int(world)
        a, s = c_size_t(), c_size_t()
        check(lib.af_ctx_workspace_bytes(h, byref(a), byref(s)), "af_ctx_workspace_bytes")
        self.accum_bytes, self.scratch_bytes = a.value, s.value
        self.device = device
        self.accum = self.scratch = None
        self._rec_host = None
        self._event = None
        if bind:
            self.bind(device)

    # -- setup -------------------------------------------------------------------
    def shard_of(self, f):
        """This rank's element range [begin, end) with f POOL blocks frozen."""
        b, e = ctypes.c_int64(), ctypes.c_int64()
        check(lib.af_ctx_shard_of(self._h, int(f), byref(b), byref(e)), "af_ctx_shard_of")
        return b.value, e.value

    def info(self):
        i = L.AfInfo()
        check(lib.af_ctx_info(self._h, byref(i)), "af_ctx_info")
        return dict(n_segments=i.n_segments, n_pool=i.n_pool, rank=i.rank, world=i.world,
                    n_total=i.n_total, shard_begin=i.shard_begin, shard_end=i.shard_end,
                    n_tiles=i.n_tiles, tile_elems=i.tile_elems, n_tiles_acc=i.n_tiles_acc,
                    tile_elems_acc=i.tile_elems_acc, n_fin_ctas=i.n_fin_ctas, n_fin_chunks=i.n_fin_chunks,
                    first_tile_of_pool=list(i.first_tile_of_pool[:i.n_pool + 1]))

    def bind(self, device=None):
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        with torch.cuda.device(dev):
            # zeroed so that never-accumulated (frozen-from-the-start) elements read as 0
            self.accum = torch.zeros(max(1, self.accum_bytes), dtype=torch.uint8, device=dev)
            self.scratch = torch.empty(self.scratch_bytes, dtype=torch.uint8, device=dev)
            check(lib.af_ctx_bind(self._h, c_void_p(self.accum.data_ptr() if self.accum_bytes else 0),
                                  c_void_p(self.scratch.data_ptr())), "af_ctx_bind")
        self._rec_host = torch.empty(ctypes.sizeof(L.AfDecision), dtype=torch.uint8, pin_memory=True)
        self._event = torch.cuda.Event()

    def set_comm(self, group=None):
        """Collective: create the library's NCCL communicator (rank 0 makes the id,
        torch.distributed broadcasts it over `group`)."""
        if self.world == 1:  # a one-rank communicator needs no bootstrap (AF_DEBUG_FORCE_NCCL tests)
            buf = (ctypes.c_uint8 * 128)()
            check(lib.af_nccl_unique_id(buf), "af_nccl_unique_id")
            uid = bytes(buf)
        else:
            uid = bootstrap_nccl_id(self.rank, group, self.device)
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        with torch.cuda.device(self.device):
            check(lib.af_ctx_set_comm(self._h, buf), "af_ctx_set_comm")

    def set_peers_local(self, peers):
        """Register every rank's context living in this process (ranks sharing one
        GPU, or single-process multi-GPU with peer access) for the NVLink one-shot
        exchange."""
        arr = (c_void_p * len(peers))(*[p._h.value for p in peers])
        check(lib.af_ctx_set_peers_local(self._h, arr), "af_ctx_set_peers_local")

    def set_peers_ipc(self, group=None):
        """Collective: exchange CUDA IPC handles of every rank's exchange buffers
        through torch.distributed and register them (one-shot NVLink exchange).
        Returns True on every rank, or False on every rank (no peers registered)
        when any rank could not export or map a handle -- fall back to set_comm()."""
        import torch.distributed as dist
        h = (ctypes.c_uint8 * L.AF_IPC_HANDLE_BYTES)()
        with torch.cuda.device(self.device):
            mine = bytes(h) if lib.af_ctx_exchange_ipc_handle(self._h, h) == L.AF_OK else None
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        ok = all(x is not None for x in allh)
        if ok:
            buf = (ctypes.c_uint8 * (L.AF_IPC_HANDLE_BYTES * self.world)).from_buffer_copy(b"".join(allh))
            with torch.cuda.device(self.device):
                ok = lib.af_ctx_set_peers_ipc(self._h, buf) == L.AF_OK
        oks = [None] * self.world
        dist.all_gather_object(oks, ok, group=group)
        if not all(oks):
            lib.af_ctx_clear_peers(self._h)
            return False
        return True

    def set_max_ctas(self, n):
        """Cap the streaming kernels' CTAs (0: the full persistent grid)."""
        check(lib.af_ctx_set_max_ctas(self._h, int(n)), "af_ctx_set_max_ctas")

    def set_grad_peers_local(self, grads):
        """NEXT 1 (ZeRO form): register every rank's full gradient buffer, for ranks
        living in this process; grads[r] is rank r's tensor."""
        for r, g in enumerate(grads):
            _dev_tensor(g, f"grads[{r}]", None, dtypes=_GRAD_TORCH[self.grad_dtype], min_numel=self.offsets[-1])
        self._rs_grads = list(grads)                 # keep the buffers alive
        arr = (c_void_p * len(grads))(*[g.data_ptr() for g in grads])
        check(lib.af_ctx_set_grad_peers_local(self._h, arr), "af_ctx_set_grad_peers_local")

    def set_grad_peers_ipc(self, grad, group=None):
        """NEXT 1 (ZeRO form), collective: export this rank's persistent gradient
        buffer, all-gather the CUDA IPC handles and map every rank's buffer."""
        import torch.distributed as dist
        self._grad(grad)
        self._rs_grads = [grad]
        h = (ctypes.c_uint8 * L.AF_IPC_HANDLE_BYTES)()
        with torch.cuda.device(self.device):
            check(lib.af_ctx_grad_ipc_handle(self._h, c_void_p(grad.data_ptr()), h), "af_ctx_grad_ipc_handle")
        allh = [None] * self.world
        dist.all_gather_object(allh, bytes(h), group=group)
        buf = (ctypes.c_uint8 * (L.AF_IPC_HANDLE_BYTES * self.world)).from_buffer_copy(b"".join(allh))
        with torch.cuda.device(self.device):
            check(lib.af_ctx_set_grad_peers_ipc(self._h, buf), "af_ctx_set_grad_peers_ipc")

    def reduce_scatter_step(self, out=None, scale=None, interval_end=False, dry_run=False, stream=None,
                            copy_record=True):
        """af_reduce_scatter_step: this rank's shard of (sum over ranks of the
        registered gradients) * scale (default 1/world) into `out` (fp32, indexed
        from shard_begin; None: not written), accumulated into Delta -- or, with
        interval_end=True, the whole interval end and decision."""
        if out is not None:
            _dev_tensor(out, "out", self.device, dtypes=(torch.float32,), min_numel=self._shard_len())
        sc = (1.0 / self.world) if scale is None else float(scale)
        flags = (L.AF_INTERVAL_END if interval_end else 0) | (L.AF_DRY_RUN if dry_run else 0)
        rec = c_void_p(self._rec_host.data_ptr()) if (copy_record and interval_end) else c_void_p(0)
        check(lib.af_reduce_scatter_step(self._h, ctypes.c_float(sc), c_void_p(out.data_ptr() if out is not None else 0),
                                         flags, rec, _stream_handle(stream)), "af_reduce_scatter_step")
        if interval_end and copy_record and not torch.cuda.is_current_stream_capturing():
            self._event.record(stream if stream is not None else torch.cuda.current_stream())
        return out

    def reduce_scatter_adamw_step(self, params, exp_avg, exp_avg_sq, lr, step, beta1=0.9, beta2=0.999, eps=1e-8,
                                  weight_decay=0.0, out=None, scale=None, interval_end=False, dry_run=False,
                                  stream=None, copy_record=True):
        """af_reduce_scatter_adamw_step: the fused reduce-scatter with AdamW on this
        rank's shard of params / exp_avg / exp_avg_sq (full flat fp32 tensors)."""
        for t, nm in ((params, "params"), (exp_avg, "exp_avg"), (exp_avg_sq, "exp_avg_sq")):
            self._f32_full(t, nm)
        if out is not None:
            _dev_tensor(out, "out", self.device, dtypes=(torch.float32,), min_numel=self._shard_len())
        sc = (1.0 / self.world) if scale is None else float(scale)
        hp = L.AfAdamW(float(lr), float(beta1), float(beta2), float(eps), float(weight_decay), int(step))
        flags = (L.AF_INTERVAL_END if interval_end else 0) | (L.AF_DRY_RUN if dry_run else 0)
        rec = c_void_p(self._rec_host.data_ptr()) if (copy_record and interval_end) else c_void_p(0)
        check(lib.af_reduce_scatter_adamw_step(
            self._h, ctypes.c_float(sc), c_void_p(params.data_ptr()), c_void_p(exp_avg.data_ptr()),
            c_void_p(exp_avg_sq.data_ptr()), byref(hp), c_void_p(out.data_ptr() if out is not None else 0), flags,
            rec, _stream_handle(stream)), "af_reduce_scatter_adamw_step")
        if interval_end and copy_record and not torch.cuda.is_current_stream_capturing():
            self._event.record(stream if stream is not None else torch.cuda.current_stream())
        return out

    def _shard_len(self):
        b, e = self.shard_of(0)
        return e - b

    def read_record(self, interval):
        """af_ctx_read_record (synchronous): the device ring's record of `interval`
        (the last 16 intervals), for callers that enqueue several intervals
        without reading each record."""
        r = L.AfDecision()
        check(lib.af_ctx_read_record(self._h, int(interval), byref(r)), "af_ctx_read_record")
        return decision_to_dict(r, self.n_segments)

    def set_debug(self, key, value):
        """af_ctx_set_debug: test / diagnostic knobs (include/af.h): AF_DEBUG_TAIL_DELAY_NS,
        AF_DEBUG_PEERS_ARRIVED, AF_DEBUG_UNSTAGED_TAIL, AF_DEBUG_FORCE_NCCL."""
        check(lib.af_ctx_set_debug(self._h, int(key), int(value)), "af_ctx_set_debug")

    def exchange_rows(self):
        """float64 view [world, L] of the exchange matrix inside the scratch buffer."""
        p = c_void_p()
        check(lib.af_ctx_exchange_rows(self._h, byref(p)), "af_ctx_exchange_rows")
        off = p.value - self.scratch.data_ptr()
        n = self.world * self.n_segments * 8
        return self.scratch[off:off + n].view(torch.float64).view(self.world, self.n_segments)

    # -- argument checks -----------------------------------------------------------
    def _grad(self, grad, name="grad"):
        return _dev_tensor(grad, name, self.device, dtypes=_GRAD_TORCH[self.grad_dtype], min_numel=self.offsets[-1])

    def _f32_full(self, t, name):
        return _dev_tensor(t, name, self.device, dtypes=(torch.float32,), min_numel=self.offsets[-1])

    # -- the hot path --------------------------------------------------------------
    def layer_norms(self, grad, interval_end=False, dry_run=False, stream=None):
        self._grad(grad)
        flags = (L.AF_INTERVAL_END if interval_end else 0) | (L.AF_DRY_RUN if dry_run else 0)
        check(lib.af_layer_norms(self._h, c_void_p(grad.data_ptr()), flags, _stream_handle(stream)),
              "af_layer_norms")

    def update_and_decide(self, dry_run=False, stream=None, copy_record=True):
        flags = L.AF_DRY_RUN if dry_run else 0
        out = c_void_p(self._rec_host.data_ptr()) if copy_record else c_void_p(0)
        check(lib.af_update_and_decide(self._h, flags, out, _stream_handle(stream)), "af_update_and_decide")
        if copy_record and not torch.cuda.is_current_stream_capturing():
            self._event.record(stream if stream is not None else torch.cuda.current_stream())

    def interval_end(self, grad, dry_run=False, stream=None, copy_record=True):
        """af_interval_end: the interval-end step and the decision in one call
        (one kernel launch when world == 1)."""
        self._grad(grad)
        flags = L.AF_DRY_RUN if dry_run else 0
        out = c_void_p(self._rec_host.data_ptr()) if copy_record else c_void_p(0)
        check(lib.af_interval_end(self._h, c_void_p(grad.data_ptr()), flags, out, _stream_handle(stream)),
              "af_interval_end")
        if copy_record and not torch.cuda.is_current_stream_capturing():
            self._event.record(stream if stream is not None else torch.cuda.current_stream())

    def adamw_step(self, params, exp_avg, exp_avg_sq, grad, lr, step, beta1=0.9, beta2=0.999, eps=1e-8,
                   weight_decay=0.0, interval_end=False, dry_run=False, stream=None, copy_record=True):
        """af_adamw_step: AdamW on this rank's shard fused with the Delta accumulate
        (or, with interval_end=True, with the whole interval end and decision)."""
        self._grad(grad)
        for t, nm in ((params, "params"), (exp_avg, "exp_avg"), (exp_avg_sq, "exp_avg_sq")):
            self._f32_full(t, nm)
        hp = L.AfAdamW(float(lr), float(beta1), float(beta2), float(eps), float(weight_decay), int(step))
        flags = (L.AF_INTERVAL_END if interval_end else 0) | (L.AF_DRY_RUN if dry_run else 0)
        out = c_void_p(self._rec_host.data_ptr()) if (copy_record and interval_end) else c_void_p(0)
        check(lib.af_adamw_step(self._h, c_void_p(params.data_ptr()), c_void_p(exp_avg.data_ptr()),
                                c_void_p(exp_avg_sq.data_ptr()), c_void_p(grad.data_ptr()), byref(hp), flags, out,
                                _stream_handle(stream)), "af_adamw_step")
        if interval_end and copy_record and not torch.cuda.is_current_stream_capturing():
            self._event.record(stream if stream is not None else torch.cuda.current_stream())

    def decision(self):
        """The last copied decision record (waits for the stream to reach it)."""
        self._event.synchronize()
        rec = L.AfDecision.from_address(self._rec_host.data_ptr())
        return decision_to_dict(rec, self.n_segments)

    def get_state(self):
        n = c_size_t()
        check(lib.af_get_state(self._h, None, byref(n)), "af_get_state")
        buf = ctypes.create_string_buffer(n.value)
        check(lib.af_get_state(self._h, buf, byref(n)), "af_get_state")
        return buf.raw[:n.value]

    def set_state(self, blob):
        buf = ctypes.create_string_buffer(blob, len(blob))
        check(lib.af_set_state(self._h, buf, len(blob)), "af_set_state")

    def close(self):
        if getattr(self, "_h", None):
            lib.af_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ActivationCache:
    """af_cache: the Storage Manager's cache of frozen-prefix outputs for this
    rank's ids (§3.2, P:335 partition by id mod world).

    Direct-mapped in HBM by default (room for every owned id).  With
    hbm_rows/host_rows it is tiered with admission (af_cache_set_capacity): room
    for I = hbm_rows + host_rows (+ disk_rows) records, the host part in
    page-locked memory, the disk part in a file (af_cache_set_disk_tier; a
    temporary file unless disk_path is given, deleted on close); puts of new ids
    beyond I are dropped (drop-newest)."""

    def __init__(self, num_examples, row_bytes, rank=0, world=1, device=None, bind=True,
                 hbm_rows=None, host_rows=0, disk_rows=0, stage_rows=256, disk_path=None):
        h = c_void_p()
        check(lib.af_cache_create(int(num_examples), int(row_bytes), int(rank), int(world), byref(h)),
              "af_cache_create")
        self._h = h
        self.num_examples, self.row_bytes, self.rank, self.world = int(num_examples), int(row_bytes), rank, world
        self.tiered = hbm_rows is not None or host_rows
        self._tmp_disk = None
        if self.tiered or disk_rows:
            self.tiered = True
            check(lib.af_cache_set_capacity(h, int(hbm_rows or 0), int(host_rows)), "af_cache_set_capacity")
        if disk_rows:
            if disk_path is None:
                import tempfile
                fd, disk_path = tempfile.mkstemp(prefix="af_cache_disk_", suffix=".bin")
                os.close(fd)
                self._tmp_disk = disk_path
            check(lib.af_cache_set_disk_tier(h, int(disk_rows), int(stage_rows), str(disk_path).encode()),
                  "af_cache_set_disk_tier")
        self.disk_path = disk_path
        p, m, hb = c_size_t(), c_size_t(), c_size_t()
        check(lib.af_cache_storage_bytes(h, byref(p), byref(m)), "af_cache_storage_bytes")
        check(lib.af_cache_host_bytes(h, byref(hb)), "af_cache_host_bytes")
        self.payload_bytes, self.meta_bytes, self.host_bytes = p.value, m.value, hb.value
        sb = c_size_t()
        check(lib.af_cache_disk_stage_bytes(h, byref(sb)), "af_cache_disk_stage_bytes")
        self.stage_bytes = sb.value
        self.payload = self.meta = self.host_tier = self.disk_stage = None
        self.device = None
        if bind:
            self.bind(device)

    def bind(self, device=None):
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        with torch.cuda.device(dev):
            self.payload = torch.empty(max(16, self.payload_bytes), dtype=torch.uint8, device=dev)
            self.meta = torch.empty(self.meta_bytes, dtype=torch.uint8, device=dev)
            check(lib.af_cache_bind(self._h, c_void_p(self.payload.data_ptr()), c_void_p(self.meta.data_ptr())),
                  "af_cache_bind")
            if self.host_bytes:
                self.host_tier = torch.empty(self.host_bytes, dtype=torch.uint8, pin_memory=True)
                check(lib.af_cache_bind_host(self._h, c_void_p(self.host_tier.data_ptr())), "af_cache_bind_host")
            if self.stage_bytes:
                # page-locked staging of the disk tier; pinned tensors are 256-byte aligned
                self.disk_stage = torch.empty(self.stage_bytes, dtype=torch.uint8, pin_memory=True)
                check(lib.af_cache_bind_disk_stage(self._h, c_void_p(self.disk_stage.data_ptr())),
                      "af_cache_bind_disk_stage")

    def _ids(self, ids):
        return _dev_tensor(ids, "ids", self.device, dtypes=(torch.int64,))

    def _rows(self, rows, n, name):
        return _dev_tensor(rows, name, self.device, min_bytes=n * self.row_bytes)

    def _depth_out(self, d, n):
        return _dev_tensor(d, "depth_out", self.device, dtypes=(torch.int32,), min_numel=n)

    def put(self, ids, rows, depth, stream=None):
        n = int(self._ids(ids).numel())
        self._rows(rows, n, "rows")
        check(lib.af_cache_put(self._h, c_void_p(ids.data_ptr()), n, c_void_p(rows.data_ptr()), int(depth),
                               _stream_handle(stream)), "af_cache_put")

    def get(self, ids, cur_boundary, rows_out, depth_out, stream=None, overlap_prev=False):
        """overlap_prev: AF_CACHE_OVERLAP_PREV -- the copy may start while the kernel
        before it on the stream finishes (the caller guarantees that kernel does not
        touch ids, this store or the outputs; see include/af.h)."""
        n = int(self._ids(ids).numel())
        self._rows(rows_out, n, "rows_out")
        self._depth_out(depth_out, n)
        check(lib.af_cache_get_ex(self._h, c_void_p(ids.data_ptr()), n, int(cur_boundary),
                                  c_void_p(rows_out.data_ptr()), c_void_p(depth_out.data_ptr()),
                                  L.AF_CACHE_OVERLAP_PREV if overlap_prev else 0, _stream_handle(stream)),
              "af_cache_get_ex")

    def get_async(self, ids, cur_boundary, rows_out, depth_out, stream):
        """Prefetch (the paper's reader process, Fig. 8): enqueue the get on a side
        stream and return an event the consumer stream waits on."""
        self.get(ids, cur_boundary, rows_out, depth_out, stream=stream)
        ev = torch.cuda.Event()
        ev.record(stream)
        return ev

    def set_peers_local(self, peers):
        """NEXT 4: register every rank's cache living in this process."""
        arr = (c_void_p * len(peers))(*[p._h.value for p in peers])
        check(lib.af_cache_set_peers_local(self._h, arr), "af_cache_set_peers_local")

    def set_peers_ipc(self, group=None):
        """NEXT 4, collective: exchange CUDA IPC handles of every rank's store."""
        import torch.distributed as dist
        h = (ctypes.c_uint8 * L.AF_CACHE_IPC_HANDLE_BYTES)()
        with torch.cuda.device(self.device):
            check(lib.af_cache_exchange_ipc_handle(self._h, h), "af_cache_exchange_ipc_handle")
        allh = [None] * self.world
        dist.all_gather_object(allh, bytes(h), group=group)
        buf = (ctypes.c_uint8 * (L.AF_CACHE_IPC_HANDLE_BYTES * self.world)).from_buffer_copy(b"".join(allh))
        with torch.cuda.device(self.device):
            check(lib.af_cache_set_peers_ipc(self._h, buf), "af_cache_set_peers_ipc")

    def get_gemm(self, ids, cur_boundary, weight, y, depth_out, rows_per_record, stream=None):
        """af_cache_get_gemm (NEXT 4): y[i] = record_i @ weight.T for the hits, the
        records read by the GEMM's TMA loads straight from the store (no batch
        copy); weight is a bf16 [N, K] tensor (torch Linear layout), y bf16
        [n * rows_per_record, N]; misses leave y untouched (depth_out = -1)."""
        n = int(self._ids(ids).numel())
        _dev_tensor(weight, "weight", self.device, dtypes=(torch.bfloat16,))
        if weight.dim() != 2:
            raise ValueError("weight must be [N, K]")
        N, K = weight.shape
        _dev_tensor(y, "y", self.device, dtypes=(torch.bfloat16,), min_numel=n * rows_per_record * N)
        self._depth_out(depth_out, n)
        check(lib.af_cache_get_gemm(self._h, c_void_p(ids.data_ptr()), n, int(cur_boundary), int(rows_per_record),
                                    int(K), c_void_p(weight.data_ptr()), int(N), c_void_p(y.data_ptr()),
                                    c_void_p(depth_out.data_ptr()), _stream_handle(stream)), "af_cache_get_gemm")

    def put_global(self, ids, rows, depth, stream=None):
        self._rows(rows, int(self._ids(ids).numel()), "rows")
        check(lib.af_cache_put_global(self._h, c_void_p(ids.data_ptr()), int(ids.numel()),
                                      c_void_p(rows.data_ptr()), int(depth), _stream_handle(stream)),
              "af_cache_put_global")

    def get_global(self, ids, cur_boundary, rows_out, depth_out, stream=None):
        n = int(self._ids(ids).numel())
        self._rows(rows_out, n, "rows_out")
        self._depth_out(depth_out, n)
        check(lib.af_cache_get_global(self._h, c_void_p(ids.data_ptr()), int(ids.numel()), int(cur_boundary),
                                      c_void_p(rows_out.data_ptr()), c_void_p(depth_out.data_ptr()),
                                      _stream_handle(stream)), "af_cache_get_global")

    def status(self):
        e, v = c_uint32(), c_int64()
        check(lib.af_cache_status(self._h, byref(e), byref(v)), "af_cache_status")
        return e.value, v.value

    def stats(self):
        i = L.AfCacheInfo()
        check(lib.af_cache_stats(self._h, byref(i)), "af_cache_stats")
        return {k: getattr(i, k) for k, _ in L.AfCacheInfo._fields_ if k != "pad"}

    def close(self):
        if getattr(self, "_h", None):
            lib.af_cache_destroy(self._h)
            self._h = None
        if getattr(self, "_tmp_disk", None):
            try:
                os.remove(self._tmp_disk)
            except OSError:
                pass
            self._tmp_disk = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def calibrate_read_seconds(row_bytes, batch_rows, device=None, reps=10):
    """Measured time to read one cached batch (af_cache_get of batch_rows hits) on
    this device: the t_batch_read of the cache-vs-recompute rule (PAPER.md:230-235:
    "few iterations of training can indicate how many layers ... need to be frozen
    before caching becomes advantageous")."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    c = ActivationCache(batch_rows, row_bytes, device=dev)
    ids = torch.arange(batch_rows, device=dev, dtype=torch.int64)
    rows = torch.zeros((batch_rows, row_bytes), dtype=torch.uint8, device=dev)
    out = torch.empty_like(rows)
    dep = torch.empty(batch_rows, dtype=torch.int32, device=dev)
    c.put(ids, rows, 1)
    c.get(ids, 1, out, dep)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        c.get(ids, 1, out, dep)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def calibrate_forward_seconds(layer_forward, iters=5, warmup=2, stream=None):
    """Measured time of one layer's forward pass (`layer_forward()`, the caller's
    callable running one frozen block on one batch) on the current stream: the
    t_layer_fwd of the cache-vs-recompute rule, taken over a few iterations of
    training ("few iterations of training can indicate how many layers
    ... need to be frozen before caching becomes advantageous"). Median of
    `iters` CUDA-event-timed calls after `warmup`."""
    s = stream if stream is not None else torch.cuda.current_stream()
    for _ in range(warmup):
        layer_forward()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        layer_forward()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


def calibrate_should_cache(layer_forward, row_bytes, batch_rows, max_layers, device=None, iters=5):
    """Both sides of the P:230-235 trade-off measured on this device: t_layer_fwd
    from a few timed forward passes of one block (`layer_forward`) and
    t_batch_read from timed cache gets of one batch; returns the smallest frozen
    depth k <= max_layers at which af_should_cache(k, t_fwd, t_read) says caching
    pays (None if none does) with the two times."""
    t_fwd = calibrate_forward_seconds(layer_forward, iters=iters)
    t_read = calibrate_read_seconds(row_bytes, batch_rows, device=device, reps=iters)
    k = next((k for k in range(1, int(max_layers) + 1) if should_cache(k, t_fwd, t_read)), None)
    return {"min_frozen_layers": k, "t_layer_fwd_s": t_fwd, "t_batch_read_s": t_read}


def bootstrap_nccl_id(rank, group=None, device=None):
    """Rank 0 creates a 128-byte ncclUniqueId through the library; torch.distributed
    broadcasts it to every rank of `group` (gloo: CPU tensor, nccl: device tensor)."""
    import torch.distributed as dist
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        buf = (ctypes.c_uint8 * 128)()
        check(lib.af_nccl_unique_id(buf), "af_nccl_unique_id")
        uid = torch.frombuffer(bytearray(bytes(buf)), dtype=torch.uint8).clone()
    if dist.get_backend(group) == "nccl":
        t = uid.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()))
        dist.broadcast(t, src=0, group=group)
        uid = t.cpu()
    else:
        dist.broadcast(uid, src=0, group=group)
    return bytes(uid.tolist())


def should_cache(frozen_layers, t_layer_fwd_s, t_batch_read_s):
    """PAPER.md:230-235 §3.2 cache-vs-recompute rule, evaluated by the library."""
    return bool(lib.af_should_cache(int(frozen_layers), float(t_layer_fwd_s), float(t_batch_read_s)))
