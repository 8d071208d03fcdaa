#!/usr/bin/env python
"""bench.py — DSG-NLM throughput on the B200 (BASELINE.json metric).

Workload (one "step"): one adaptive DSG-NLM denoise of the config-4 image —
8192 x 8192 float32 seeded scene + noise 25/255, search 21x21 (R=10), patch
7x7 Gaussian sigma_p=2, h=12/255 (bandwidth h/sqrt(2)); the full pipeline
(sweep A, rs, sweep B, fixups, max, finalize).  Every N runs the row-strip
algorithm (parallel.ShardedDSG): N = 1 is one strip (exchanges are no-ops;
the product call dsg_nlm_denoise on the same image is timed beside it as
"single_call"), N > 1 (torchrun) shards the rows across the ranks (NCCL
halo / partial-block exchange, max all-reduce); the problem size is fixed
("strong" scaling).

value    = 8192^2 * 441 pixel-offsets / device time per step (max over
           ranks), in Gpixel*offset/s, inputs resident in HBM (268 MB > L2,
           so every step streams from HBM; no flush needed);
e2e      = the same through the public API with host buffers, transfers in
           the timed region: the headline is the reference's own call shape,
           dsg_nlm_denoise(float64 numpy) -> float64 numpy; the pipelined
           DenoiseStream and the synchronous pinned-tensor call beside it;
roofline = the dominant kernel of the step (CUDA events on the library
           stream): the fused sweep A (FP32-bound: SURVEY.md §8(d)'s algorithmic
           ops per pixel-offset / its launch time vs the FFMA rate measured on
           this GPU by pnp_peak_rates) or the k-cache stream of sweep B
           (HBM-bound: 4 B per half-window pair vs MEASURED_PEAKS hbm_gbs); plus
           "denoise": the whole step vs the FP32 roofline of the algorithm
           (20.95 ops per pixel-offset);
cpu_baseline = the reference itself (pnprestore installed unmodified into
           oracle/_ref) on one uncached crop of the same image, 1 core.
Extras: config 5 (64 x 1024^2 SR ADMM, 20 iterations) split image-per-GPU
at every N; at N = 1 also config 1 (256^2 denoise) and ADMM iterations/s for
configs 2 and 3, each with the reference's final PSNR beside ours
(tests/golden).

``--impl reference`` times the reference's own dsg_nlm_denoise (oracle/_ref)
with all host cores, one process per core, on uncached crops of the same
image.  ``--dist-backend gloo`` runs N > 1 with host-staged messages (ranks
may share a GPU: tests the N > 1 path on one device).
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

H_C4 = 8192
R_C4, P_C4, SIGMA_P, H_BW = 10, 7, 2.0, 12 / 255
OPS_PER_UNIT_ADAPTIVE = (4 * P_C4 + 14) * ((21 * 21 - 1) / 2) / (21 * 21)   # 20.95
MUFU_PER_UNIT_ADAPTIVE = 2 * ((21 * 21 - 1) / 2) / (21 * 21)                # 0.998
METRIC = "DSG-NLM Gpixel*offset/s (config 4: 8192^2, R=10, P=7 Gaussian)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pnp", choices=["pnp", "reference"])
    ap.add_argument("--size", type=int, default=H_C4, help="image side (default: config 4)")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / cpu / ADMM extras")
    ap.add_argument("--no-cache", action="store_true",
                    help="disable the k cache (recompute the patch filter in sweep B)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N > 1: NCCL between GPUs, or gloo with host-staged messages "
                         "(several ranks sharing one GPU, for testing the N > 1 path)")
    return ap.parse_args()


# --------------------------------------------------------------------------- helpers

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self):
        if self.proc is None or not getattr(self, "lines", None):
            return None
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def committed_traffic() -> dict:
    """Per-launch dram bytes of the sweep kernels from the committed ncu capture."""
    try:
        d = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
        return {k: v["dram_bytes_per_launch"] for k, v in d["kernels"].items()}
    except Exception:
        return {}


def measured_hbm_gbs() -> float:
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def _synth():
    """paper_1901_06110_b200/synth.py loaded by path: numpy only, so the
    reference arm never imports the package (or maps libpnpb200.so)."""
    mod = sys.modules.get("_pnp_synth")
    if mod is None:
        import importlib.util
        spec = importlib.util.spec_from_file_location(
            "_pnp_synth", ROOT / "paper_1901_06110_b200" / "synth.py")
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        sys.modules["_pnp_synth"] = mod
    return mod


def make_image_rows(n: int, r0: int, r1: int) -> np.ndarray:
    """Rows [r0, r1) of the config-4 input (float32), generated independently."""
    synth = _synth()
    clean = synth.scene(n, n, 4, rows=(r0, r1))
    return synth.noisy(clean, 25 / 255, 5, first_index=r0 * n).astype(np.float32)


def reference_crops(band: np.ndarray, side: int, count: int, seed: int):
    """`count` seeded side x side crops of a band of config-4 rows (float32)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        r = int(rng.integers(0, band.shape[0] - side + 1))
        c = int(rng.integers(0, band.shape[1] - side + 1))
        out.append(np.ascontiguousarray(band[r:r + side, c:c + side]))
    return out


# --------------------------------------------------------------------------- reference arm

def _repo_so_mapped():
    """Shared objects of this repo mapped into this process (must be none in
    the reference arm)."""
    try:
        maps = Path("/proc/self/maps").read_text()
    except OSError:
        return None
    root = str(ROOT)
    return sorted({ln.split()[-1] for ln in maps.splitlines()
                   if ln.split()[-1].startswith(root) and ".so" in ln.split()[-1]})


def run_reference(args, rank, world):
    """The reference's own dsg_nlm_denoise (oracle/_ref = /root/reference/pkg
    installed unmodified; box patch weights, its SAT distance engine) on all
    host cores, one process per core, each step one uncached crop per
    process (crops larger than KERNEL_CACHE_BYTES allows, as the full
    8192^2 image is)."""
    if rank != 0:
        return
    import multiprocessing as mp

    from oracle import refcpu
    n = args.size
    bw = H_BW / math.sqrt(2.0)
    cores = os.cpu_count() or 1
    workers = max(1, min(cores, 64))
    side = refcpu.uncached_side(R_C4)
    per_step, total_units = [], 0
    band = make_image_rows(n, 0, min(n, 2 * side))  # input generation is not timed
    with mp.get_context("spawn").Pool(workers) as pool:
        warm = reference_crops(band, 64, workers, 1)
        for _ in range(args.warmup):  # spawn / imports / page-in only
            pool.map(refcpu.denoise_job, [(c, P_C4, R_C4, bw) for c in warm])
        for i in range(args.steps):
            jobs = [(c, P_C4, R_C4, bw) for c in reference_crops(band, side, workers, 100 + i)]
            t = time.perf_counter()
            res = pool.map(refcpu.denoise_job, jobs)
            per_step.append(time.perf_counter() - t)
            total_units += sum(u for u, _ in res)
    sec = sum(per_step)
    value = total_units / sec / 1e9
    sample = (f"each step: {workers} processes x one {side}x{side} crop of the config-4 image "
              f"(largest side whose kernel maps exceed KERNEL_CACHE_BYTES, so the reference "
              f"recomputes them per sweep as at 8192^2), pnprestore.dsg_nlm_denoise as shipped "
              f"(box patch weights: the reference has no Gaussian mode), float64")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gpixel*offset/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded scene + noise)",
        "config": {"workload": "config 4 DSG-NLM (sampled crops)", "image": f"{n}x{n}",
                   "crop": f"{side}x{side}", "R": R_C4, "P": P_C4, "sigma_p": None,
                   "h": H_BW},
        "cpu_baseline": {"value": value, "unit": "Gpixel*offset/s", "cores": workers,
                         "kind": refcpu.kind(), "sample": sample},
        "e2e": {"value": value, "unit": "Gpixel*offset/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "repo_so_mapped": _repo_so_mapped(),
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm

def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1901_06110_b200 as pnp
    from paper_1901_06110_b200 import profiling

    # (--dist-backend gloo may put several ranks on one GPU)
    local_rank = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if args.no_cache:
        profiling.set_cache_limit(0, local_rank)
    n = args.size
    params = pnp.PatchParams.from_h(P_C4, R_C4, H_BW, SIGMA_P)
    units = n * n * (2 * R_C4 + 1) ** 2

    def barrier():
        if world > 1:
            dist.barrier()

    # every N (1 included) runs the row-strip algorithm (parallel.ShardedDSG):
    # the scaling curve compares one code path; at N = 1 there is one strip
    # and the exchanges are no-ops (same kernels as dsg_nlm_denoise, which is
    # timed beside it as "single_call")
    from paper_1901_06110_b200.parallel import HostStagedComm, LocalComm, ShardedDSG, TorchComm
    if world == 1:
        comm = LocalComm()
    elif args.dist_backend == "gloo":
        comm = HostStagedComm()
    else:
        comm = TorchComm()
    sh = ShardedDSG(params, n, n, world, [rank], comm, device=dev, kcache=not args.no_cache)
    st = sh.states[0]
    y0, y1 = st.lay.rows
    st.own(st.buf).copy_(torch.from_numpy(make_image_rows(n, y0, y1)))

    def step():
        sh.denoise()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    profiling.enable(True, local_rank)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        barrier()
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        barrier()
    prof = profiling.read(local_rank)
    profiling.enable(False, local_rank)
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t[0])
    value = units / (ms_max * 1e-3) / 1e9

    launches = sum(v[1] for v in prof.values())
    peak_ffma, peak_ex2 = profiling.peak_rates(local_rank)
    nominal = torch.cuda.get_device_properties(dev).multi_processor_count * 128 * 1.965e9
    hbm_peak = measured_hbm_gbs()
    units_rank = units / world * args.steps          # pixel-offsets swept by this rank
    sweep_ms, sweep_n = prof["sweep"]
    cached_ms, cached_n = prof["sweep_cached"]
    traffic = committed_traffic()
    # algorithmic FP32 ops per pixel-offset of the recompute sweeps:
    # sweep A (mass) (F+5)*N+/(2R+1)^2, sweep B (F+9)*N+/(2R+1)^2 with F = 2P
    half = ((2 * R_C4 + 1) ** 2 - 1) / 2 / (2 * R_C4 + 1) ** 2
    ops_a, ops_b = (2 * P_C4 + 5) * half, (2 * P_C4 + 9) * half
    ops_unit = ops_a + (ops_b if cached_n == 0 else 0.0)
    kbytes_unit = 4.0 * half  # k cache: one float per pixel and half-window offset
    kernels = []
    if sweep_ms > 0:
        ach = ops_unit * units_rank / (sweep_ms * 1e-3) / 1e12
        name = "dsg_sweep_kernel<7,10,1,STORE>" if cached_n else "dsg_sweep_kernel<7,10,C,RECOMPUTE>"
        kernels.append({
            "kernel": name, "role": "sweep A (mass) + k-cache store" if cached_n
            else "sweep A + sweep B, fused recompute",
            "bound": "fp32", "achieved": ach, "peak": peak_ffma / 1e12, "unit": "Top/s",
            "frac": ach / (peak_ffma / 1e12), "frac_of_nominal": ach / (nominal / 1e12),
            "ops_per_pixel_offset": ops_unit, "ms_per_step": sweep_ms / args.steps,
            "launches_per_step": sweep_n / args.steps,
            "sfu_frac": (half * (1 if cached_n else 2)) * units_rank / (sweep_ms * 1e-3) / peak_ex2,
            "hbm_write_GBps": (kbytes_unit * units_rank / (sweep_ms * 1e-3) / 1e9) if cached_n else 0.0,
            "traffic": traffic.get("sweep_store" if cached_n else "sweep_recompute")})
    if cached_n:
        ach = kbytes_unit * units_rank / (cached_ms * 1e-3) / 1e9
        kernels.append({
            "kernel": "dsg_sweep_kernel<7,10,2,CACHED>", "role": "sweep B over the k cache "
            "(bulk async copies into SMEM, mbarrier double buffer)", "bound": "hbm",
            "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
            "bytes_per_pixel_offset": kbytes_unit, "ms_per_step": cached_ms / args.steps,
            "launches_per_step": cached_n / args.steps, "traffic": traffic.get("sweep_cached")})
    dom = max(kernels, key=lambda k: k["ms_per_step"]) if kernels else None
    roofline = {k: v for k, v in (dom or {}).items()}
    # the whole denoise against the FP32 roofline of the algorithm (north star)
    roof_rate = peak_ffma / ((ops_a + ops_b))  # pixel-offsets / s at 100% FFMA
    roofline.update({
        "peak_source": "fp32: FFMA rate measured by pnp_peak_rates on this GPU (nominal "
                       f"148x128x1965MHz = {nominal / 1e12:.2f} Top/s); hbm: MEASURED_PEAKS.json",
        "share_of_step": (dom["ms_per_step"] / ms) if dom else None,
        "kernels": kernels,
        "ex2_peak_per_s": peak_ex2,
        "denoise": {"pixel_offsets_per_s": value * 1e9,
                    "fp32_roofline_pixel_offsets_per_s": roof_rate,
                    "frac": value * 1e9 / roof_rate,
                    "ops_per_pixel_offset": ops_a + ops_b,
                    "note": "whole adaptive denoise (all kernels) vs the FFMA roofline of the "
                            "two-sweep algorithm (SURVEY §8(d): 20.95 FP32 ops per pixel-offset)"},
        "traffic_note": "dram read+write bytes per launch from the committed ncu --set full "
                        "capture (profiles/ncu_traffic.json)",
    })
    line = {
        "metric": METRIC, "value": value, "unit": "Gpixel*offset/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded rectangle/disc/gradient scene + splitmix noise 25/255)",
        "config": {"workload": "config 4: adaptive DSG-NLM of one 8192x8192 image"
                               if n == H_C4 else f"config-4 parameters at {n}x{n}",
                   "image": f"{n}x{n}", "R": R_C4, "P": P_C4, "sigma_p": SIGMA_P, "h": H_BW,
                   "parallelism": f"row-strips x{world}" if world > 1 else "single GPU",
                   "l2": "inputs 268 MB > 126 MB L2 (no flush needed)"},
        "roofline": roofline, "gpu_launches": launches, "impl": "pnp",
    }
    clocks = clk.summary()
    line["clocks"] = clocks
    if world == 1:
        # the product call on the same image, timed beside the strip path
        x = st.own(st.buf).clone()
        del sh, st
        torch.cuda.empty_cache()
        for _ in range(2):
            pnp.dsg_nlm_denoise(x, params)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            pnp.dsg_nlm_denoise(x, params)
        e1.record()
        torch.cuda.synchronize()
        ms1 = e0.elapsed_time(e1) / args.steps
        line["single_call"] = {"value": units / (ms1 * 1e-3) / 1e9, "ms_per_step": ms1,
                               "api": "paper_1901_06110_b200.dsg_nlm_denoise(device tensor)"}
        del x
        torch.cuda.empty_cache()

    if not args.no_extras:
        # e2e through the public API with pinned host buffers: every step
        # uploads its image, denoises and downloads the result (DenoiseStream:
        # H2D / compute / D2H on three streams, overlapped across steps)
        if world == 1:
            host_in = torch.from_numpy(make_image_rows(n, 0, n)).pin_memory()
            stream = pnp.DenoiseStream(params, (n, n))
            host_outs = [torch.empty_like(host_in).pin_memory() for _ in range(2)]
            nbytes = host_in.numel() * 4
            stream.run([host_in] * 2, host_outs)  # warm-up
            torch.cuda.synchronize()
            barrier()
            e0.record()
            stream.run([host_in] * args.steps, [host_outs[i % 2] for i in range(args.steps)])
            e1.record()
            torch.cuda.synchronize()
            t_stream = e0.elapsed_time(e1) / args.steps
            ref_out = pnp.dsg_nlm_denoise(host_in.to(dev), params).cpu()
            assert torch.equal(host_outs[(args.steps - 1) % 2], ref_out), "stream != denoise"
            # the stream's k cache was allocated on its compute stream: hand it
            # back so the calls below (current stream) reuse one block
            torch.cuda.empty_cache()

            def e2e_step():  # the synchronous single-image call, reported beside it
                xd = host_in.to(dev, non_blocking=True)
                yd = pnp.dsg_nlm_denoise(xd, params)
                host_outs[0].copy_(yd, non_blocking=True)
        else:
            own = torch.from_numpy(make_image_rows(n, y0, y1)).pin_memory()
            host_out = torch.empty_like(own).pin_memory()

            def e2e_step():
                st.own(st.buf).copy_(own, non_blocking=True)
                sh.denoise()
                host_out.copy_(st.own(st.out), non_blocking=True)
            nbytes = own.numel() * 4
        for _ in range(max(1, args.warmup // 2)):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        e0.record()
        for _ in range(args.steps):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if world == 1:
            # headline: the reference's own call shape -- float64 numpy in, new
            # float64 numpy out (validation, casts and both transfers included)
            img64 = host_in.numpy().astype(np.float64)
            out64 = pnp.dsg_nlm_denoise(img64, params)  # warm-up
            assert np.array_equal(out64, ref_out.numpy().astype(np.float64)), "numpy != denoise"
            walls = []
            for _ in range(max(3, args.steps)):
                w0 = time.perf_counter()
                pnp.dsg_nlm_denoise(img64, params)
                walls.append((time.perf_counter() - w0) * 1e3)
            ms_np = float(np.median(walls))
            line["e2e"] = {
                "value": units / (ms_np * 1e-3) / 1e9, "unit": "Gpixel*offset/s",
                "ms_per_step": ms_np, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                "api": "paper_1901_06110_b200.dsg_nlm_denoise(float64 numpy) -> float64 numpy, "
                       "the reference's call shape (host cast + banded upload overlapping sweep "
                       "A, banded download + float64 cast); median wall time of the synchronous "
                       "call",
                "stream": {"value": units / (t_stream * 1e-3) / 1e9, "ms_per_step": t_stream,
                           "api": "paper_1901_06110_b200.DenoiseStream.run(pinned host "
                                  "float32 images): per step H2D + dsg_nlm_denoise + D2H, "
                                  "overlapped across steps on 3 streams"},
                "sync_call": {"value": units / (float(t[0]) * 1e-3) / 1e9,
                              "ms_per_step": float(t[0]),
                              "api": "pinned float32 host -> device copy, dsg_nlm_denoise, "
                                     "device -> pinned host copy, one image at a time"}}
        else:
            line["e2e"] = {"value": units / (float(t[0]) * 1e-3) / 1e9, "unit": "Gpixel*offset/s",
                           "h2d_bytes_per_step": nbytes * world,
                           "d2h_bytes_per_step": nbytes * world, "ms_per_step": float(t[0]),
                           "api": "parallel.ShardedDSG.denoise"}
        if world > 1:
            del sh, st
        torch.cuda.empty_cache()  # the k caches (59 GB at 8192^2) sit in torch's cache
        line["config5"] = config5(pnp, dev, rank, world, True)
        if rank == 0 and world == 1:
            line["admm"] = admm_extras(pnp, dev)
            from oracle import refcpu  # the checker / baseline, timed on the host only
            side = refcpu.uncached_side(R_C4)
            band = make_image_rows(n, 0, min(n, 2 * side))
            (crop,) = reference_crops(band, side, 1, 7)
            c0 = time.process_time()
            cu, wall = refcpu.denoise_job((crop, P_C4, R_C4, params.bandwidth))
            cpu = time.process_time() - c0
            line["cpu_baseline"] = {
                "value": cu / wall / 1e9, "unit": "Gpixel*offset/s", "cores": 1,
                "kind": refcpu.kind(),
                "sample": f"one {side}x{side} crop of the config-4 image (uncached: its kernel "
                          "maps exceed KERNEL_CACHE_BYTES, as at 8192^2) through "
                          "pnprestore.dsg_nlm_denoise as shipped (oracle/_ref; box patch "
                          "weights, SAT distances), float64, 1 thread",
                "wall_s": wall, "cpu_s": cpu, "host_cores_available": os.cpu_count()}
    if rank == 0:
        print(json.dumps(line), flush=True)


def bicubic_x2(y32: np.ndarray) -> np.ndarray:
    """Bicubic x2 guide of an observation, float64 on the host, clipped,
    float32 (tests/golden/make_golden_configs.py's recipe)."""
    import torch
    import torch.nn.functional as F
    t = torch.from_numpy(y32.astype(np.float64))
    g = F.interpolate(t[None, None], scale_factor=2, mode="bicubic", align_corners=False)[0, 0]
    return g.clamp(0, 1).numpy().astype(np.float32)


def golden_check(name, v, recs, y=None, image=None):
    """The reference's own result for this run (tests/golden/, produced by
    pnprestore here): final PSNR beside ours, max |dv|."""
    try:
        gd = np.load(ROOT / "tests" / "golden" / name)
    except OSError:
        return {}
    ps = [float(np.atleast_1d(r.psnr)[image or 0]) for r in recs]
    vv = v.double().cpu().numpy() if hasattr(v, "cpu") else np.asarray(v, np.float64)
    out = {"psnr_oracle_db": float(gd["rec"][-1, 3]), "psnr_gpu_db": ps[-1],
           "psnr_diff_db": ps[-1] - float(gd["rec"][-1, 3]),
           "max_abs_dv_vs_oracle": float(np.abs(vv - gd["v"]).max()),
           "oracle": f"tests/golden/{name} (pnprestore linearized_pnp_admm, float64)"}
    if y is not None:
        # the observation is simulated here on the device (fp32 blur, float64
        # noise), the golden's by the reference in float64: same seeds, equal
        # to fp32 rounding (not bitwise)
        yy = y.double().cpu().numpy() if hasattr(y, "cpu") else np.asarray(y, np.float64)
        out["inputs_max_abs_diff_vs_golden"] = float(np.abs(yy - gd["y"].astype(np.float64)).max())
    return out


def admm_extras(pnp, dev):
    """Configs 1, 2, 3 and 5 on the device: denoise time, ADMM iterations/s,
    final PSNR beside the reference's (tests/golden)."""
    import torch

    from paper_1901_06110_b200 import synth
    res = {}
    # config 1 (the reference's CPU-runnable case): one 256^2 image, radius 5,
    # patch 5 Gaussian sigma_p 1.5, h = 10/255, noise 20/255; W x and row sums d
    img1 = torch.from_numpy(synth.noisy(synth.scene(256, 256, 1), 20 / 255, 2).astype(np.float32))
    img1 = img1.to(dev)
    p1 = pnp.PatchParams.from_h(5, 5, 10 / 255, 1.5)
    for _ in range(3):
        pnp.dsg_nlm_denoise(img1, p1, return_aux=True)
    torch.cuda.synchronize()
    e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_a.record()
    for _ in range(50):
        pnp.dsg_nlm_denoise(img1, p1, return_aux=True)
    e_b.record()
    torch.cuda.synchronize()
    ms1 = e_a.elapsed_time(e_b) / 50
    res["config1_denoise_256"] = {"ms_per_denoise": ms1,
                                  "gpixel_offsets_per_s": 256 * 256 * 121 / (ms1 * 1e-3) / 1e9,
                                  "reference_cpu_note": "survey: pnprestore 0.31 s on 1 CPU core"}
    # config 2: 512^2 SR, blur 9x9 sigma 1 symmetric, x2, noise 5/255, 30 its, frozen bicubic guide
    truth = synth.scene(512, 512, 2).astype(np.float32)
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    y = pnp.sr_simulate(truth.astype(np.float64), op, 5 / 255, seed=102).astype(np.float32)
    yd = torch.from_numpy(y).to(dev)
    guide = torch.from_numpy(bicubic_x2(y)).to(dev)
    p2 = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=30, constraint=pnp.UNIT_BOX)
    gt = torch.from_numpy(truth).to(dev)
    prob_c2 = pnp.make_sr_problem(op, yd, ground_truth=gt)
    runs = []
    for i in range(6):  # first run warms up; median of the others
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fz = pnp.freeze_guide(guide, p2)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        v, recs = pnp.linearized_pnp_admm(prob_c2, cfg, denoiser=fz.as_denoiser())
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if i:
            runs.append((t2 - t1, t1 - t0))
    solve_s = float(np.median([r[0] for r in runs]))
    freeze_s = float(np.median([r[1] for r in runs]))
    res["config2_sr_512"] = {"iters": 30, "iters_per_s": 30 / solve_s,
                             "freeze_ms": freeze_s * 1e3,
                             "end_to_end_ms": (solve_s + freeze_s) * 1e3,
                             "device_ms": recs[-1].time_ms, "psnr_db": recs[-1].psnr,
                             **golden_check("cfg2.npz", v, recs, y=y),
                             "timing": "median of 5 solves (linearized_pnp_admm call, wall)"}
    # paper Fig. 2: the standard PnP-ADMM (exact x-update by CG, native
    # batched solver) on the same problem and denoiser
    cfg_s = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=30,
                             constraint=pnp.UNIT_BOX, cg_tol=1e-6, cg_max_iters=200)
    prob2 = pnp.make_sr_problem(op, yd, ground_truth=gt)
    for _ in range(2):
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        vs, recs_s = pnp.standard_pnp_admm_cg(prob2, cfg_s, denoiser=fz.as_denoiser())
        torch.cuda.synchronize()
        t4 = time.perf_counter()
    res["config2_standard_cg"] = {"iters": 30, "iters_per_s": 30 / (t4 - t3),
                                  "psnr_db": recs_s[-1].psnr,
                                  "linearized_speedup": (t4 - t3) / solve_s}
    # config 3: 512^2 QIS, K = 4x4x8 = 128 jots, alpha_s = 8 -> gain 64, 50 its, dsg-fixed @15
    truth3 = synth.scene(512, 512, 3).astype(np.float32)
    model = pnp.QisModel(128, 64.0)
    counts = pnp.qis_simulate(truth3.astype(np.float64), model, seed=103)
    prob = pnp.make_qis_problem(counts, model, ground_truth=torch.from_numpy(truth3).to(dev))
    prob.x0 = torch.from_numpy(prob.x0.astype(np.float32)).to(dev)
    cfg3 = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=pnp.default_qis_alpha(counts, model),
                            max_iters=50, freeze_at=15, constraint=pnp.UNIT_BOX,
                            denoiser="dsg-fixed", patch_side=7, window_radius=10,
                            bandwidth=(10 / 255) / math.sqrt(2), patch_sigma=2.0)
    runs = []
    gc.collect()
    gc.disable()  # host-timed solves: no collector pauses inside
    try:
        for i in range(15):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            v, recs = pnp.linearized_pnp_admm(prob, cfg3)
            torch.cuda.synchronize()
            if i >= 3:
                runs.append(time.perf_counter() - t0)
    finally:
        gc.enable()
    res["config3_qis_512"] = {"iters": 50, "iters_per_s": 50 / float(np.median(runs)),
                              "psnr_db": recs[-1].psnr,
                              **golden_check("cfg3.npz", v, recs),
                              "timing": "median of 12 solves (wall) incl. the freeze at "
                                        "iteration 15, after 3 untimed"}
    res["reference_cpu_note"] = "survey: pnprestore config-2 shape 0.79 iters/s on 1 CPU core"
    return res


def config5(pnp, dev, rank, world, dist_ok):
    """Config 5: 64 independent 1024^2 SR problems, 20 iterations, frozen
    bicubic guides, per-image alpha; split image-per-GPU (rank r solves images
    [64 r / N, 64 (r+1) / N) as one batched call: blockIdx.z).  Solve time per
    rank from CUDA events (median of 3 after one untimed), max over ranks."""
    import torch
    import torch.distributed as dist
    synth = _synth()
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    p2 = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
    nb, side = 64, 1024
    i0, i1 = nb * rank // world, nb * (rank + 1) // world
    mine = list(range(i0, i1))
    truths, ys = [], []
    for i in mine:  # the golden's recipe: float64 simulation, float32 observation
        t_i = synth.scene(side, side, 1000 + i).astype(np.float32)
        truths.append(t_i)
        ys.append(pnp.sr_simulate(t_i.astype(np.float64), op, 5 / 255,
                                  seed=1100 + i).astype(np.float32))
    yb = torch.from_numpy(np.stack(ys)).to(dev)
    gtb = torch.from_numpy(np.stack(truths)).to(dev)
    guides = torch.from_numpy(np.stack([bicubic_x2(y_i) for y_i in ys])).to(dev)
    cfg5 = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=20, constraint=pnp.UNIT_BOX)
    prob5 = pnp.make_sr_problem(op, yb, ground_truth=gtb)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fz5 = None
    for _ in range(2):  # the second freeze is timed (the first warms the pool)
        fz5 = None
        torch.cuda.synchronize()
        e0.record()
        fz5 = pnp.freeze_guide(guides, p2)
        e1.record()
        torch.cuda.synchronize()
        t_freeze = e0.elapsed_time(e1) / 1e3
    runs = []
    for i in range(4):
        torch.cuda.synchronize()
        e0.record()
        v5, recs5 = pnp.linearized_pnp_admm(prob5, cfg5, denoiser=fz5.as_denoiser())
        e1.record()
        torch.cuda.synchronize()
        if i:
            runs.append(e0.elapsed_time(e1) / 1e3)
    t = torch.tensor([float(np.median(runs)), t_freeze], device=dev, dtype=torch.float64)
    if world > 1 and dist_ok:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_solve, t_freeze = float(t[0]), float(t[1])
    kc5 = fz5.cache_info()
    fz5 = None
    res = {
        "images": nb, "iters": 20, "n_gpus": world, "images_per_gpu": len(mine),
        "image_iters_per_s": nb * 20 / t_solve,
        "pixel_offsets_per_s_in_applies": nb * side * side * 441 * 20 / t_solve,
        "freeze_ms": t_freeze * 1e3, "end_to_end_ms": (t_freeze + t_solve) * 1e3,
        "kcache_rows_cached": f"{kc5['rows_cached']}/{kc5['tile_rows']}",
        "psnr_db_mean_rank0": float(np.mean(recs5[-1].psnr)),
        "scaling": "strong (64 images split image-per-GPU, no collective on the data path)",
        "timing": "per-rank CUDA events: median of 3 solves after one untimed, max over ranks; "
                  "freeze timed separately"}
    res["oracle_images"] = {f"img{i}": golden_check(f"cfg5_img{i}.npz", v5[j], recs5, y=ys[j],
                                                    image=j)
                            for j, i in enumerate(mine) if i in (0, 63)}
    return res


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "pnp" and args.dist_backend == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
