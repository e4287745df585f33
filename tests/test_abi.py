"""C-ABI tests that need no GPU: the library loads, exports exactly what
include/af.h declares, validates arguments synchronously, and computes its
host-side shard / tile tables correctly."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2102_01386_b200 as af
from paper_2102_01386_b200 import _lib as L
from afinputs import bert_layout, tiny_layout, uniform_layout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "af.h")


def declared_symbols():
    src = open(HEADER).read()
    return set(re.findall(r"^AF_API\s+[\w\s\*]+?\b(af_\w+)\(", src, flags=re.M))


def test_library_exports_every_declared_symbol():
    decl = declared_symbols()
    assert len(decl) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", af.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert decl <= exported, decl - exported
    assert {s for s in exported if s.startswith("af_")} == decl  # nothing undeclared leaks
    assert decl == set(L.SIGNATURES), decl ^ set(L.SIGNATURES)


def test_struct_sizes_match_header_layout():
    assert ctypes.sizeof(L.AfDecision) == 4 * 4 + 8 + 4 + 4 + 3 * 8 * 256
    assert ctypes.sizeof(L.AfConfig) == 40


def test_status_strings_and_version():
    assert L.lib.af_status_str(L.AF_EINVAL) == b"AF_EINVAL"
    assert L.lib.af_version() == b"0.1.0"


def test_should_cache_printed_examples(golden):
    for k, tf, tr, want in golden("spec_examples.json")["should_cache"]["cases"]:
        assert af.should_cache(k, tf, tr) == want


def _create(offsets, kinds, dt=L.AF_DT_F32, **cfg):
    offs = (ctypes.c_int64 * len(offsets))(*offsets)
    knd = (ctypes.c_int32 * max(1, len(kinds)))(*kinds)
    lay = L.AfLayout(len(kinds), offs, knd, dt)
    c = dict(percentile=50.0, pct_method=0, acc_mode=0, tie_rel_eps=1e-5, min_active=2, rank=0, world=1)
    c.update(cfg)
    conf = L.AfConfig(c["percentile"], c["pct_method"], c["acc_mode"], c["tie_rel_eps"], c["min_active"],
                      c["rank"], c["world"])
    h = ctypes.c_void_p()
    st = L.lib.af_ctx_create(ctypes.byref(lay), ctypes.byref(conf), ctypes.byref(h))
    if st == L.AF_OK:
        L.lib.af_ctx_destroy(h)
    return st


@pytest.mark.parametrize("offsets,kinds,cfg", [
    ([0, 10], [1], {}),
    ([0, 5, 10, 20], [0, 1, 2], {}),
    ([0, 5, 10, 20], [1, 1, 1], dict(percentile=100.0, pct_method=1, acc_mode=1, world=8, rank=7)),
])
def test_create_accepts_valid(offsets, kinds, cfg):
    assert _create(offsets, kinds, **cfg) == L.AF_OK


@pytest.mark.parametrize("offsets,kinds,cfg", [
    ([0, 10], [0], {}),                        # no POOL
    ([1, 10], [1], {}),                        # offsets[0] != 0
    ([0, 10, 10], [1, 1], {}),                 # not strictly increasing
    ([0, 5, 10], [1, 0], {}),                  # PRE after POOL
    ([0, 5, 10, 15], [1, 2, 1], {}),           # POOL after HEAD
    ([0, 5, 10], [1, 3], {}),                  # bad kind
    ([0, 10], [1], dict(percentile=0.0)),
    ([0, 10], [1], dict(percentile=100.5)),
    ([0, 10], [1], dict(percentile=float("nan"))),
    ([0, 10], [1], dict(pct_method=7)),
    ([0, 10], [1], dict(acc_mode=2)),
    ([0, 10], [1], dict(min_active=0)),
    ([0, 10], [1], dict(tie_rel_eps=-1.0)),
    ([0, 10], [1], dict(world=0)),
    ([0, 10], [1], dict(world=2, rank=2)),
    ([0, 10], [1], dict(world=65)),
])
def test_create_rejects_invalid(offsets, kinds, cfg):
    assert _create(offsets, kinds, **cfg) == L.AF_EINVAL


def test_create_rejects_too_many_segments_and_bad_dtype():
    offs = list(range(0, 258))
    assert _create(offs, [1] * 257) == L.AF_EINVAL
    assert _create([0, 10], [1], dt=5) == L.AF_EINVAL


def test_null_arguments():
    assert L.lib.af_ctx_create(None, None, None) == L.AF_EINVAL
    assert L.lib.af_layer_norms(None, None, 0, None) == L.AF_EINVAL
    assert L.lib.af_update_and_decide(None, 0, None, None) == L.AF_EINVAL
    assert L.lib.af_cache_create(10, 64, 0, 1, None) == L.AF_EINVAL


def _expected_tiles(lay, sb, se, tile_elems, big_mult=1, big_frac_pct=0, upto_seg=None):
    """Independent re-count of the segment-aligned tiles (tapered for the
    interval-end table: big_mult x tiles in the first big_frac_pct % of the shard)."""
    n = 0
    big_until = sb + (se - sb) // 100 * big_frac_pct
    for l in range(lay.n_segments if upto_seg is None else upto_seg):
        lo, hi = max(lay.offsets[l], sb), min(lay.offsets[l + 1], se)
        pos = lo
        while pos < hi:
            te = tile_elems * big_mult if pos < big_until else tile_elems
            pos = min(hi, (pos // te + 1) * te)
            n += 1
    return n


@pytest.mark.parametrize("which,dt", [("base", "bf16"), ("large", "f32"), ("base", "f32")])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shards_cover_buffer_and_tiles_are_segment_aligned(which, dt, world):
    lay = bert_layout(which)
    prev_end = 0
    total_tiles = 0
    for r in range(world):
        fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt, rank=r, world=world, bind=False)
        i = fm.info()
        assert i["shard_begin"] == prev_end
        assert i["shard_begin"] % 8 == 0
        prev_end = i["shard_end"]
        assert i["tile_elems"] % 8 == 0 and i["tile_elems"] >= 4096
        assert i["n_tiles"] == _expected_tiles(lay, i["shard_begin"], i["shard_end"], i["tile_elems"], 1, 85)
        assert i["n_tiles_acc"] == _expected_tiles(lay, i["shard_begin"], i["shard_end"], i["tile_elems_acc"])
        assert fm.accum_bytes == 4 * (i["shard_end"] - i["shard_begin"])
        ft = i["first_tile_of_pool"]
        assert ft == sorted(ft) and ft[0] == 0
        total_tiles += i["n_tiles"]
        # balanced within one shard-alignment unit
        assert abs((i["shard_end"] - i["shard_begin"]) - lay.n / world) <= 8
        fm.close()
    assert prev_end == lay.n


@pytest.mark.parametrize("which,dt", [("base", "bf16"), ("large", "f32")])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_active_suffix_shards_balance_every_boundary(which, dt, world):
    """shard_active: for every boundary f the ranks' shards tile the active suffix
    [A_f, n) (A_f = start of the first unfrozen segment; PRE goes with block 0)
    contiguously, balanced within one alignment unit; Delta is full size; the
    largest per-f table is reported; the fused AdamW / reduce-scatter refuse."""
    lay = bert_layout(which)
    pool = [l for l, k in enumerate(lay.kinds) if k == 1]
    fms = [af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt, rank=r, world=world, bind=False,
                             shard_active=True) for r in range(world)]
    te = fms[0].info()["tile_elems"]
    for f in range(len(pool) + 1):
        A = lay.offsets[pool[f]] if f < len(pool) else lay.offsets[pool[-1] + 1]
        if f == 0:
            A = 0
        prev = A
        for fm in fms:
            b, e = fm.shard_of(f)
            assert b == prev and (b == A or b % 8 == 0)
            assert abs((e - b) - (lay.n - A) / world) <= 8
            prev = e
        assert prev == lay.n
    for r, fm in enumerate(fms):
        i = fm.info()
        assert (i["shard_begin"], i["shard_end"]) == fm.shard_of(0)
        assert fm.accum_bytes == 4 * lay.n
        assert i["n_tiles"] == max(_expected_tiles(lay, *fm.shard_of(f), te, 1, 85) for f in range(len(pool) + 1))
        # the static shards are unchanged by the option at world 1
    one = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt, bind=False, shard_active=True)
    assert one.shard_of(5) == (0, lay.n) and one.accum_bytes == 4 * lay.n
    for fm in fms:
        fm.close()


def test_active_suffix_shards_refuse_fused_optimizer_paths():
    lay = tiny_layout()
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32", rank=0, world=2, bind=False,
                           shard_active=True)
    import ctypes as C
    hp = L.AfAdamW(1e-3, 0.9, 0.999, 1e-8, 0.0, 1)
    assert L.lib.af_adamw_step(fm._h, None, None, None, None, C.byref(hp), 0, None, None) == L.AF_ESTATE
    assert L.lib.af_reduce_scatter_step(fm._h, C.c_float(1.0), None, 0, None, None) == L.AF_ESTATE
    fm.close()


def test_first_tile_skips_embedding_with_first_block():
    lay = bert_layout("base")
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="bf16", bind=False)
    i = fm.info()
    te = i["tile_elems"]
    # f = 1 frozen: PRE and POOL[0] skipped
    assert i["first_tile_of_pool"][1] == _expected_tiles(lay, 0, lay.n, te, 1, 85, upto_seg=2)
    assert i["first_tile_of_pool"][2] == _expected_tiles(lay, 0, lay.n, te, 1, 85, upto_seg=3)
    assert i["first_tile_of_pool"][0] == 0


def test_step_sumsq_needs_no_accumulator():
    lay = tiny_layout()
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32", acc_mode="step_sumsq", bind=False)
    assert fm.accum_bytes == 0


def test_unbound_calls_report_workspace():
    lay = uniform_layout(1 << 12, 4)
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32", bind=False)
    buf = (ctypes.c_float * 16)()
    assert L.lib.af_layer_norms(fm._h, ctypes.addressof(buf) // 16 * 16 + 16, 1, None) == L.AF_EWORKSPACE
    assert L.lib.af_update_and_decide(fm._h, 0, None, None) == L.AF_EWORKSPACE


def test_debug_knob_and_ring_read_host_checks():
    lay = uniform_layout(1 << 12, 4)
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32", bind=False)
    assert L.lib.af_ctx_set_debug(fm._h, L.AF_DEBUG_TAIL_DELAY_NS, 1000) == L.AF_OK
    assert L.lib.af_ctx_set_debug(fm._h, L.AF_DEBUG_TAIL_DELAY_NS, -1) == L.AF_EINVAL
    assert L.lib.af_ctx_set_debug(fm._h, L.AF_DEBUG_TAIL_DELAY_NS, 2 * 10 ** 9) == L.AF_EINVAL
    assert L.lib.af_ctx_set_debug(fm._h, L.AF_DEBUG_UNSTAGED_TAIL, 1) == L.AF_OK
    assert L.lib.af_ctx_set_debug(fm._h, L.AF_DEBUG_UNSTAGED_TAIL, 2) == L.AF_EINVAL
    assert L.lib.af_ctx_set_debug(fm._h, L.AF_DEBUG_FORCE_NCCL, 0) == L.AF_OK
    assert L.lib.af_ctx_set_debug(fm._h, L.AF_DEBUG_FORCE_NCCL, -1) == L.AF_EINVAL
    assert L.lib.af_ctx_set_debug(fm._h, 99, 0) == L.AF_EINVAL
    assert L.lib.af_ctx_set_debug(None, L.AF_DEBUG_TAIL_DELAY_NS, 0) == L.AF_EINVAL
    rec = L.AfDecision()
    assert L.lib.af_ctx_read_record(fm._h, 0, ctypes.byref(rec)) == L.AF_EWORKSPACE
    assert L.lib.af_ctx_read_record(fm._h, 0, None) == L.AF_EINVAL
    fm.close()


def test_binding_validates_tensors_before_the_abi():
    # the ABI sees raw pointers only: the binding refuses wrong dtype / size /
    # layout / device before any call (out-of-bounds device access)
    import torch
    lay = uniform_layout(1 << 12, 4)
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32", bind=False)
    with pytest.raises(ValueError):
        fm.layer_norms(torch.zeros(lay.n))                      # host tensor
    c = af.ActivationCache(100, 64, bind=False)
    with pytest.raises(ValueError):
        c.put(torch.zeros(3, dtype=torch.int64), torch.zeros((3, 64), dtype=torch.uint8), 1)
    fm.close()
    c.close()


def test_disk_tier_host_checks(tmp_path):
    h = ctypes.c_void_p()
    assert L.lib.af_cache_create(1000, 64, 0, 1, ctypes.byref(h)) == L.AF_OK
    path = str(tmp_path / "tier.bin").encode()
    assert L.lib.af_cache_set_disk_tier(h, 10, 8, path) == L.AF_ESTATE        # needs a tiered store first
    assert L.lib.af_cache_set_capacity(h, 5, 5) == L.AF_OK
    assert L.lib.af_cache_set_disk_tier(h, 0, 8, path) == L.AF_EINVAL
    assert L.lib.af_cache_set_disk_tier(h, 10, 0, path) == L.AF_EINVAL
    assert L.lib.af_cache_set_disk_tier(h, 10, 8, b"/nonexistent-dir/x") == L.AF_EINVAL
    assert L.lib.af_cache_set_disk_tier(h, 10, 8, path) == L.AF_OK
    assert L.lib.af_cache_set_disk_tier(h, 10, 8, path) == L.AF_ESTATE        # once
    assert os.path.getsize(tmp_path / "tier.bin") == 10 * 64
    sb = ctypes.c_size_t()
    assert L.lib.af_cache_disk_stage_bytes(h, ctypes.byref(sb)) == L.AF_OK
    assert sb.value >= 8 * 64 + 10 * 4 and sb.value % 256 == 8 * 64 % 256
    assert L.lib.af_cache_bind_disk_stage(h, None) == L.AF_EINVAL
    info = L.AfCacheInfo()
    assert L.lib.af_cache_stats(h, ctypes.byref(info)) == L.AF_EWORKSPACE    # not bound
    assert L.lib.af_cache_destroy(h) == L.AF_OK


def test_cache_get_gemm_host_checks():
    h = ctypes.c_void_p()
    assert L.lib.af_cache_create(100, 128 * 64 * 2, 0, 1, ctypes.byref(h)) == L.AF_OK
    buf = (ctypes.c_uint8 * 64)()
    a = ctypes.addressof(buf) // 16 * 16 + 16
    assert L.lib.af_cache_get_gemm(None, a, 1, 0, 128, 64, a, 32, a, a, None) == L.AF_EINVAL
    assert L.lib.af_cache_get_gemm(h, a, 1, 0, 128, 64, a, 32, a, a, None) == L.AF_EWORKSPACE   # not bound
    assert L.lib.af_cache_get_gemm(h, a, 0, 0, 128, 64, a, 32, a, a, None) == L.AF_EWORKSPACE
    L.lib.af_cache_destroy(h)


def test_reduce_scatter_host_checks():
    # NEXT 1 (ZeRO form): argument / state errors are synchronous host checks
    lay = uniform_layout(1 << 12, 4)
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32", rank=0, world=2, bind=False)
    assert L.lib.af_reduce_scatter_step(None, 1.0, None, 0, None, None) == L.AF_EINVAL
    assert L.lib.af_reduce_scatter_step(fm._h, 0.5, None, 0, None, None) == L.AF_EWORKSPACE
    assert L.lib.af_ctx_set_grad_peers_local(fm._h, None) == L.AF_EINVAL
    assert L.lib.af_ctx_grad_ipc_handle(fm._h, None, None) == L.AF_EINVAL
    assert L.lib.af_ctx_set_max_ctas(fm._h, -1) == L.AF_EINVAL
    assert L.lib.af_ctx_set_max_ctas(fm._h, 0) == L.AF_OK
    hp = L.AfAdamW(1e-3, 0.9, 0.999, 1e-8, 0.0, 0)           # step 0: invalid
    buf = (ctypes.c_float * 16)()
    a = ctypes.addressof(buf) // 16 * 16 + 16
    assert L.lib.af_reduce_scatter_adamw_step(fm._h, 1.0, a, a, a, ctypes.byref(hp), None, 0, None,
                                              None) == L.AF_EINVAL
    fm.close()


def test_cache_create_validation_and_sizes():
    h = ctypes.c_void_p()
    assert L.lib.af_cache_create(100, 100, 0, 1, ctypes.byref(h)) == L.AF_EINVAL   # not a multiple of 16
    assert L.lib.af_cache_create(100, 64, 3, 2, ctypes.byref(h)) == L.AF_EINVAL    # rank >= world
    assert L.lib.af_cache_create(-1, 64, 0, 1, ctypes.byref(h)) == L.AF_EINVAL
    c = af.ActivationCache(100_000, 196_608, rank=3, world=8, bind=False)
    assert c.payload_bytes == 12_500 * 196_608
    assert c.meta_bytes == (256 + 12_500 * 16 + 255) // 256 * 256 + 2 * 64 * 8
    c2 = af.ActivationCache(10, 64, rank=3, world=4, bind=False)       # ids 3, 7
    assert c2.payload_bytes == 2 * 64


def test_cache_tiered_capacity_validation_and_sizes():
    c = af.ActivationCache(100_000, 196_608, rank=0, world=8, bind=False, hbm_rows=1000, host_rows=500)
    assert c.payload_bytes == 1000 * 196_608
    assert c.host_bytes == 500 * 196_608
    assert c.meta_bytes == (256 + 12_500 * 16 + (1500 + 65536) * 4 + 255) // 256 * 256 + 2 * 64 * 8
    h = ctypes.c_void_p()
    assert L.lib.af_cache_create(100, 64, 0, 1, ctypes.byref(h)) == L.AF_OK
    assert L.lib.af_cache_set_capacity(h, 0, 0) == L.AF_OK      # slots may come from a disk tier (checked at bind)
    assert L.lib.af_cache_set_capacity(h, -1, 5) == L.AF_EINVAL
    assert L.lib.af_cache_set_capacity(h, 10, 0) == L.AF_OK
    assert L.lib.af_cache_bind_host(h, None) == L.AF_EINVAL
    L.lib.af_cache_destroy(h)
