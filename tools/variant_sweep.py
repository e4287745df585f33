#!/usr/bin/env python
"""Build libautofreeze with each compile-time variant and time the streaming
kernels through bench.py (run on the GPU box).  Prints one JSON line per
(variant, workload) with the per-phase GB/s; the default build is restored at
the end.

    python tools/variant_sweep.py [--steps 200] > gpurun_out/variants.jsonl
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = {
    "default": "",
    "end_bf16_12k": "-DAF_TILE_ELEMS_BF16=12288",
    "end_bf16_24k": "-DAF_TILE_ELEMS_BF16=24576",
    "rs_bf16_u4": "-DAF_U_RS_VEC_BF16=4",
    "rs_bf16_u16": "-DAF_U_RS_VEC_BF16=16",
    "rs_end_bf16_u2": "-DAF_U_RS_VEC_END_BF16=2",
    "fin3": "-DAF_FIN_WIDE=3",
    "fin3_512": "-DAF_FIN_WIDE=3 -DAF_FIN3_CHUNK=512",
    "fin3_min512": "-DAF_FIN_WIDE=3 -DAF_FIN3_MIN_TILES=512",
    "timing_fin3": "-DAF_TIMING=1 -DAF_FIN_WIDE=3",
    "fin_narrow": "-DAF_FIN_WIDE=0",
    "fin_inkernel": "-DAF_FIN_WIDE=2",
    "acc_dnc": "-DAF_D_HINT_ACC=1",
    "st_cs": "-DAF_D_STORE=0",
    "fwd_only": "-DAF_ALTERNATE_ORDER=0",
    "p_st_wb": "-DAF_P_STORE=1",
    "acc_st_wb": "-DAF_D_STORE=1",
    "acc_st_ef": "-DAF_D_STORE=2",
    "acc_dnc_st_ef": "-DAF_D_HINT_ACC=1 -DAF_D_STORE=2",
    "acc_u4": "-DAF_U_ACC=4",
    "acc_16k": "-DAF_TILE_ACC_F32=16384 -DAF_TILE_ACC_BF16=16384",
    "ssq_old": "-DAF_TILE_SSQ_F32=8192 -DAF_TILE_SSQ_BF16=16384 -DAF_U_SSQ_F32=4 -DAF_U_SSQ_BF16=4",
    "ssq_64k_bf16": "-DAF_TILE_SSQ_BF16=65536",
    "ssq_f32_16k": "-DAF_TILE_SSQ_F32=16384",
    "timing_fin_inkernel": "-DAF_TIMING=1 -DAF_FIN_WIDE=2",
    "end8k": "-DAF_TILE_ELEMS_F32=8192 -DAF_TILE_ELEMS_BF16=8192",
    "end_f32_8k": "-DAF_TILE_ELEMS_F32=8192",
    "end_f32_4k": "-DAF_TILE_ELEMS_F32=4096",
    "end_f32_8k_bf16_32k": "-DAF_TILE_ELEMS_F32=8192 -DAF_TILE_ELEMS_BF16=32768",
    "end4k_taper4": "-DAF_TILE_ELEMS_F32=4096 -DAF_TILE_ELEMS_BF16=4096 -DAF_TILE_BIG_MULT=4",
    "end8k_taper2": "-DAF_TILE_ELEMS_F32=8192 -DAF_TILE_ELEMS_BF16=8192 -DAF_TILE_BIG_MULT=2",
    "end4k_taper4_95": "-DAF_TILE_ELEMS_F32=4096 -DAF_TILE_ELEMS_BF16=4096 -DAF_TILE_BIG_MULT=4 -DAF_TILE_BIG_FRAC_PCT=95",
    "end8k_taper4": "-DAF_TILE_ELEMS_F32=8192 -DAF_TILE_ELEMS_BF16=8192 -DAF_TILE_BIG_MULT=4",
    "acc4k_taper": "-DAF_TILE_ACC_F32=4096 -DAF_TILE_ACC_BF16=4096",
    "timing": "-DAF_TIMING=1",
    "timing_fin_narrow": "-DAF_TIMING=1 -DAF_FIN_WIDE=0",
    "taper_off": "-DAF_TILE_BIG_MULT=1",
    "taper4": "-DAF_TILE_BIG_MULT=4",
    "taper8_90": "-DAF_TILE_BIG_FRAC_PCT=90",
    "taper16": "-DAF_TILE_BIG_MULT=16",
    "c_s3_2cta": "-DAF_CACHE_STAGES=3 -DAF_CACHE_CTAS_PER_SM=2",
    "c_16k_s12": "-DAF_CACHE_CHUNK=16384 -DAF_CACHE_STAGES=12",
    "c_16k_s6_2cta": "-DAF_CACHE_CHUNK=16384 -DAF_CACHE_STAGES=6 -DAF_CACHE_CTAS_PER_SM=2",
    "c_64k_s3": "-DAF_CACHE_CHUNK=65536 -DAF_CACHE_STAGES=3",
    "tma1": "-DAF_TMA=1",
    "tma2": "-DAF_TMA=2",
    "minb3": "-DAF_MINB_END=3",
    "u2": "-DAF_U_END=2",
    "ghint0": "-DAF_G_HINT=0",
    "ghint0_minb3": "-DAF_G_HINT=0 -DAF_MINB_END=3",
    "acc4k": "-DAF_TILE_ACC_F32=4096 -DAF_TILE_ACC_BF16=4096",
    "acc16k_bf16": "-DAF_TILE_ACC_BF16=16384",
    "end8k_f32": "-DAF_TILE_ELEMS_F32=8192",
    "end32k_bf16": "-DAF_TILE_ELEMS_BF16=32768",
    "tile_bf16_32k": "-DAF_TILE_ELEMS_BF16=32768",
    "tile_bf16_8k": "-DAF_TILE_ELEMS_BF16=8192",
    "tile_f32_8k": "-DAF_TILE_ELEMS_F32=8192",
    "tile_f32_32k": "-DAF_TILE_ELEMS_F32=32768",
    "bf16_acc_u4": "-DAF_U_ACC=4",
    "g_nc": "-DAF_G_HINT=1",
    "g_nc_d_nc": "-DAF_G_HINT=1 -DAF_D_HINT_END=1",
    "g_nc_d_nc_u8": "-DAF_G_HINT=1 -DAF_D_HINT_END=1 -DAF_U_END=8",
    "g_nc_d_nc_u8_minb2": "-DAF_G_HINT=1 -DAF_D_HINT_END=1 -DAF_U_END=8 -DAF_MINB_END=2",
    "g_nc_d_nc_minb3": "-DAF_G_HINT=1 -DAF_D_HINT_END=1 -DAF_MINB_END=3",
    "g_nc_d_nc_minb4": "-DAF_G_HINT=1 -DAF_D_HINT_END=1 -DAF_MINB_END=4",
    "g_nc_acc_u2": "-DAF_G_HINT=1 -DAF_U_ACC=2",
    "g_nc_acc_u8": "-DAF_G_HINT=1 -DAF_U_ACC=8",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--cache", action="store_true", help="run tools/cache_probe.py instead of bench.py")
    ap.add_argument("--probe", help="run tools/<PROBE>.py (e.g. latency_probe, tail_probe) instead of bench.py")
    a = ap.parse_args()
    sys.path.insert(0, ROOT)
    for name, extra in VARIANTS.items():
        if a.only and name not in a.only:
            continue
        env = dict(os.environ, AF_NVCC_EXTRA=extra)
        subprocess.run([sys.executable, os.path.join(ROOT, "paper_2102_01386_b200", "_build.py"), "--force"], cwd=ROOT, env=env,
                       check=True)
        if a.cache or a.probe:
            probe = "cache_probe" if a.cache else a.probe
            r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", probe + ".py")], cwd=ROOT,
                               capture_output=True, text=True)
            for line in r.stdout.strip().splitlines():
                try:
                    print(json.dumps({"variant": name, "flags": extra, **json.loads(line)}), flush=True)
                except Exception:  # noqa: BLE001
                    print(json.dumps({"variant": name, "flags": extra, "out": line[-2000:]}), flush=True)
            if r.returncode:
                print(json.dumps({"variant": name, "err": r.stderr[-1500:]}), flush=True)
            continue
        for wl in ("bert-large-f32", "bert-base-bf16"):
            r = subprocess.run([sys.executable, "bench.py", "--workload", wl, "--steps", str(a.steps), "--warmup", "10",
                                "--no-e2e", "--no-cpu-baseline", "--no-cache-sweep", "--no-secondary"], cwd=ROOT,
                               capture_output=True, text=True)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
            except Exception:  # noqa: BLE001
                print(json.dumps({"variant": name, "workload": wl, "error": r.stderr[-2000:]}), flush=True)
                continue
            ph = d["phases"]
            print(json.dumps({"variant": name, "flags": extra, "workload": wl, "value": d["value"],
                              "ms_per_step": d["ms_per_step"],
                              "accumulate_gbs": ph["accumulate"]["gbs"], "grad_norm_gbs": ph["grad_norm_decide"]["gbs"],
                              "accumulate_ms": ph["accumulate"]["ms"], "grad_norm_ms": ph["grad_norm_decide"]["ms"],
                              "in_step_ms": {k: v["ms"] for k, v in (d.get("phases_in_step") or {}).items()
                                             if isinstance(v, dict)},
                              "adamw_gbs": (d.get("next1_fused_adamw") or {}).get("gbs"),
                              "rs_p1_gbs": (d.get("next1_fused_reduce_scatter_p1") or {}).get("gbs"),
                              "rs_p1_end_gbs": ((d.get("next1_fused_reduce_scatter_p1") or {}).get("interval_end")
                                                or {}).get("gbs"),
                              "clocks": d.get("clocks")}), flush=True)
    subprocess.run([sys.executable, os.path.join(ROOT, "paper_2102_01386_b200", "_build.py"), "--force"], cwd=ROOT, check=True)


if __name__ == "__main__":
    main()
