#!/usr/bin/env python
"""Benchmark of the MHFD hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mhfd|reference]

One *step* = one pass of the whole hot path over one
batch of synthetic EM tiles resident in HBM: percentiles -> fused stretch/blur/DoG/
argmax -> NMS + threshold + compaction -> overlap pruning -> focus scores, plus (N>1)
the NCCL all-gather of every rank's (count, score).  Workload (config C4 of
SURVEY.md §8(d)): per GPU a batch of 64 tiles of 4096x4096 u8 (image g: seed 1000+g,
defocus 0.5*(g mod 9) px, dose 300), sigma 1-10, 10 scales, tau = 0.1*dt = 0.09,
overlap 0.5.  Images are independent, so per-GPU work is fixed as N grows ("weak").
The 1.07 GB batch per GPU is larger than L2 (126 MB), so no L2 flush is needed.

Timing: W untimed warm-up steps, then exactly K steps bracketed by barrier +
cudaDeviceSynchronize and CUDA events on the launching stream; max over ranks.
Per-stage device times come from events the library records on the same stream
(mhfd_timing_*), which gives the dominant kernel's (mhfd_schedule_name) duration for
the roofline (k_tc, the tcgen05 kernel, by default).  `e2e` repeats the measurement through mhfd_focus_score_host with the
batch in pinned host memory (H2D copies and the D2H of scores inside the timed
region).  `cpu_baseline` times the oracle (oracle/, f64, plain C) on rank 0 on a
bounded sample (the tile's percentiles + a 512-row band, extrapolated to the tile) on
all host cores and on 1 thread.

`--impl reference`: the oracle IS the reference arm for this tier (there is no
reference implementation to install): rank 0 times it on the host
cores, each step the same sample as cpu_baseline; other ranks exit 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MPix/s and ms/image (4096² tile, 10 scales) at 1/2/4/8 B200 vs HBM roofline"
SIZE = 4096
E2E_CHUNK = 16   # images per host-path chunk (staging 3 x 16 x 16.8 MB)
SIGMA = (1.0, 10.0)
NSCALES = 10
TAU = 0.1 * (SIGMA[1] - SIGMA[0]) / NSCALES
OVERLAP = 0.5
# FP32 peak (SURVEY.md §8(d) "P_fp32"): nominal 148 SMs x 128 FFMA/clk x 1.965 GHz
# (clocks.max.sm) = 37.2 T FFMA/s; the FFMA microbenchmark measured 36.1 T FFMA/s
# (profiles/r01_ubench_ffma.json), reported beside it.
FP32_PEAK_TFFMA = 148 * 128 * 1.965e9 / 1e12
FP32_UBENCH_TFFMA = 36.1


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def radii():
    dt = (SIGMA[1] - SIGMA[0]) / NSCALES
    return [math.ceil(5.0 * (SIGMA[0] + i * dt)) for i in range(NSCALES + 1)]


def cascade_ffma_per_px(smin: float = SIGMA[0], smax: float = SIGMA[1], n: int = NSCALES) -> int:
    """SURVEY.md §8(d) F_alg: FFMA per pixel of the cheapest exact separable schedule at
    the parity radius k = 5 — level 1 direct (2 passes x (2R_1+1)), then each next level
    as the cascade increment sigma_inc = sqrt(t_{i+1}^2 - t_i^2) (2 x (2R_inc+1)).
    674 at C3 (sigma 1-10, n 10), 2,662 at C5 (sigma 1-30, n 20)."""
    dt = (smax - smin) / n
    t = [smin + i * dt for i in range(n + 1)]
    f = 2 * (2 * math.ceil(5.0 * t[0]) + 1)
    for i in range(1, n + 1):
        f += 2 * (2 * math.ceil(5.0 * math.sqrt(t[i] ** 2 - t[i - 1] ** 2)) + 1)
    return f


def direct_ffma_per_px(smin: float = SIGMA[0], smax: float = SIGMA[1], n: int = NSCALES) -> int:
    dt = (smax - smin) / n
    return sum(2 * (2 * math.ceil(5.0 * (smin + i * dt)) + 1) for i in range(n + 1))


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock and throttle reasons."""

    REASONS = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
               "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            log("clock sampling unavailable:", e)
            self.max = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def make_batch(rank: int, B: int, device) -> torch.Tensor:
    import synth
    imgs = torch.empty((B, SIZE, SIZE), dtype=torch.uint8, device=device)
    for b in range(B):
        g = rank * B + b
        imgs[b] = synth.em_tile(SIZE, SIZE, 1000 + g, defocus=0.5 * (g % 9), dose=300.0, device=device)
    return imgs


# ------------------------------------------------------------------ oracle timing
ORACLE_ROWS = 512   # band of one tile per oracle sample (both the cpu_baseline and the reference arm)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(img: np.ndarray, rows: int = ORACLE_ROWS) -> dict:
    """The oracle as it stands on a bounded sample of one 4096^2 tile: percentiles and
    stretch of the whole tile (t_tile), then Eq. 2 DoG / Eq. 3 NMS / pruning of a band
    of `rows` rows (t_band).  The rate extrapolates to the whole tile,
    T = t_tile + t_band * SIZE / rows, value = SIZE^2 / T (MPix/s): the tile-wide
    percentile sort is charged once per tile, not once per band (the round-1 reference
    arm charged it per band and understated the oracle ~4x)."""
    import oracle
    t0 = time.perf_counter()
    lo, hi = oracle.percentiles(img)
    f = oracle.stretch(img, lo, hi)
    t1 = time.perf_counter()
    y0 = (SIZE - rows) // 2
    D = oracle.dog_stack(f, SIGMA[0], SIGMA[1], NSCALES, rows=(y0, y0 + rows))
    cand = oracle.nms_paper(D, TAU)
    keep = oracle.prune(cand, SIGMA[0], SIGMA[1], NSCALES, OVERLAP)
    t2 = time.perf_counter()
    T = (t1 - t0) + (t2 - t1) * SIZE / rows
    return {"value": SIZE * SIZE / T / 1e6, "t_tile_s": t1 - t0, "t_band_s": t2 - t1, "rows": rows,
            "tile_s_extrapolated": T, "candidates": int(len(cand)), "kept": int(keep.sum())}


def _sample_text(r: dict, threads: int) -> str:
    return (f"tile 0 (4096^2 u8): percentiles+stretch of the tile ({r['t_tile_s']:.2f} s) + DoG/NMS/pruning "
            f"of a {r['rows']}-row band ({r['t_band_s']:.2f} s), f64, {threads} thread(s); extrapolated to the "
            f"tile: {r['tile_s_extrapolated']:.1f} s per 16.8 MPix")


def cpu_baseline(img: np.ndarray) -> dict:
    """the oracle on all host cores and on 1 thread, with the CPU model."""
    import oracle
    ncpu = os.cpu_count() or 1
    oracle.set_threads(ncpu)
    r = oracle_sample(img)
    cores = oracle.get_threads()
    oracle.set_threads(1)
    r1 = oracle_sample(img, rows=256)
    oracle.set_threads(ncpu)
    return {"value": r["value"], "unit": "MPix/s", "cores": cores, "kind": "oracle", "sample": _sample_text(r, cores),
            "cpu_model": cpu_model(), "one_thread": {"value": r1["value"], "unit": "MPix/s", "cores": 1,
                                                     "sample": _sample_text(r1, 1)},
            "candidates_in_band": r["candidates"], "kept_in_band": r["kept"]}


def run_reference(args) -> None:
    """The reference arm of this tier: the oracle as it stands on the host cores, each
    step one oracle_sample of the same workload (same sample and rate definition as
    cpu_baseline, so the two agree)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import synth
    oracle.set_threads(os.cpu_count() or 1)
    img = synth.em_tile_np(SIZE, SIZE, 1000, defocus=0.0, dose=300.0, bits=8)
    vals, last = [], None
    for k in range(args.warmup + args.steps):
        last = oracle_sample(img)
        if k >= args.warmup:
            vals.append(last["value"])
    value = statistics.median(vals)
    ms = SIZE * SIZE / (value * 1e6) * 1e3   # per 4096^2 tile
    cores = oracle.get_threads()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "MPix/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_per_image": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C4 tile (4096x4096 u8 synthetic EM, sigma 1-10, 10 scales, tau 0.09, "
                                   "overlap 0.5); each step one oracle sample of tile 0, rate extrapolated to the tile",
                       "rows_per_step": ORACLE_ROWS, "parallelism": f"{cores} host threads (OpenMP)"},
            "cpu_baseline": {"value": value, "unit": "MPix/s", "cores": cores, "kind": "oracle",
                             "sample": _sample_text(last, cores), "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "MPix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def peaks() -> tuple[dict, str]:
    """Roofline denominators: MEASURED_PEAKS.json (driver-written), else the fallback
    of B200_PROFILING.md (6.65 TB/s, 1.59 PF burst / ~1.4 PF sustained)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "of measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "of fallback (B200_PROFILING.md)"


def _ncu_summary(name: str) -> dict:
    p = os.path.join(ROOT, "profiles", f"ncu_{name}_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def roofline_of(det, B: int, kern_ms: float, step_ms: float, stage_ms: dict) -> dict:
    """Roofline per SURVEY.md §8(d).  On CUDA cores the path is FP32-ALU
    bound: F_alg = the cascade FFMA count of the cheapest exact separable schedule (674
    FFMA/px at C3), B_alg = 1 B/px.  The tcgen05 kernel k_tc beats that bound, so for it
    the top-level roofline is the tensor pipe (issued banded-GEMM work vs the burst
    cuBLAS peak) and the ALU figures move to `alu_cascade`.  For the dominant kernel (stage a2-a6,
    timed live with the library's CUDA events on the launching stream):
      achieved = F_alg x 2 FLOP x pixels per launch / kernel ms,
      peak     = nominal FP32 (148 x 128 FFMA/clk x 1.965 GHz, x 2 FLOP),
      frac     = achieved / peak = T_bound / T_meas (roofline_frac of §8(d) item 2).
    Beside it: the whole step's roofline_frac, hbm_frac from the ncu DRAM bytes (per
    kernel and for the step), and for k_tc the tensor pipe: the dense-equivalent banded
    MMA flops it issues against the BURST cuBLAS peak (k_tc runs unthrottled) next to
    ncu's tensor-active %."""
    pk, pk_note = peaks()
    name = det.schedule("u8")
    px = B * SIZE * SIZE
    f_alg = cascade_ffma_per_px()
    t_bound_ms = f_alg * px / (FP32_PEAK_TFFMA * 1e12) * 1e3
    achieved = 2 * f_alg * px / (kern_ms * 1e-3) / 1e12
    peak = 2 * FP32_PEAK_TFFMA
    ncu = _ncu_summary(name)
    traffic = ncu.get("dram_bytes_per_image", None)
    traffic = traffic * B if traffic is not None else None
    hbm_bw = pk["hbm_gbs"]
    step_bytes = ncu.get("step_dram_bytes_per_image")
    line = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": name, "kernel_ms_per_launch": kern_ms, "px_per_launch": px,
            "alg_ffma_per_px": f_alg, "alg_flops_per_px": 2 * f_alg,
            "alg_note": "SURVEY 8(d) F_alg: cascade FFMA of the cheapest exact separable schedule (level 1 direct, "
                        "then sigma_inc increments, k = 5), x 2 FLOP",
            "peak_note": "nominal FP32: 148 SMs x 128 FFMA/clk x 2 x 1.965 GHz (B200_PROFILING.md unit counts)",
            "frac_vs_ffma_ubench": achieved / (2 * FP32_UBENCH_TFFMA),
            "roofline_frac": t_bound_ms / kern_ms, "T_bound_ms": t_bound_ms, "T_meas_ms": kern_ms,
            "roofline_frac_step": t_bound_ms / step_ms, "step_ms": step_ms, "share_of_step": kern_ms / step_ms,
            "direct_ffma_per_px": direct_ffma_per_px(),
            "hbm": {"alg_bytes_per_px": 1, "peak_GBs": hbm_bw, "peak_note": pk_note,
                    "kernel_GBs": traffic / (kern_ms * 1e-3) / 1e9 if traffic else None,
                    "hbm_frac_kernel": traffic / (kern_ms * 1e-3) / 1e9 / hbm_bw if traffic else None,
                    "step_GBs": step_bytes * B / (step_ms * 1e-3) / 1e9 if step_bytes else None,
                    "hbm_frac_step": step_bytes * B / (step_ms * 1e-3) / 1e9 / hbm_bw if step_bytes else None,
                    "alg_frac_step": px / (step_ms * 1e-3) / 1e9 / hbm_bw,
                    "source": ncu.get("source")}}
    if name == "k_tc":
        # The tensor-core kernel beats the FP32 cascade bound above (roofline_frac > 1), so
        # the ALU roofline no longer bounds it: its roofline is the fp16 tensor pipe, with
        # the banded-GEMM formulation's work per pixel (DESIGN.md §6.1 / §8) as F_alg.
        fpp = det.schedule_flops_per_pixel("u8")
        t_ach = fpp * px / (kern_ms * 1e-3) / 1e12
        floor_pf = 148 * 8192 * 1.965e9 / 1e12   # tcgen05 kind::f16 M128 floor: 8192 FLOP/clk/SM at 1.965 GHz
        alu = {k: line.pop(k) for k in ("bound", "achieved", "peak", "unit", "frac")}
        alu["note"] = "method-level ALU roofline (SURVEY 8(d)): frac > 1 = faster than any FP32 cascade schedule"
        line.update({"bound": "tensor", "achieved": t_ach, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                     "frac": t_ach / pk["bf16_tflops"]})
        line["alu_cascade"] = alu
        line["tensor"] = {"alg_flops_per_px": fpp, "peak_note": "burst cuBLAS bf16 " + pk_note + " (fp16 = bf16 rate; "
                          "k_tc runs unthrottled)", "peak_sustained": pk["bf16_tflops_sustained"],
                          "frac_sustained": t_ach / pk["bf16_tflops_sustained"],
                          "peak_tcgen05_floor": floor_pf, "frac_tcgen05_floor": t_ach / floor_pf,
                          "ncu_tensor_active_pct": ncu.get("tensor_active_pct"),
                          "note": "F_alg = the banded Toeplitz MMA work the formulation issues per pixel (zeros of "
                                  "the band included; 2 row-pass and 3 column-pass fp16 products per level)"}
    return line


def other_configs(dev) -> dict:
    """The other configs of SURVEY.md §8(d), measured on rank 0 after the main step (not
    part of `value`): C2 = one 1024^2 u8 tile, host-visible latency of focus_score_host
    (H2D + compute + score on the host) and device time; C3 = the same for one 4096^2
    tile; C5 = one 8192^2 u16 tile, sigma 1-30, 20 scales (generic CUDA-core schedule),
    device time.  Median of 11 after 3 warm-ups."""
    import synth
    import paper_2108_12050_b200 as mhfd
    out = {}

    def timed(det, img_dev, img_host):
        for _ in range(3):
            det.focus_score(img_dev)
            det.focus_score_host(img_host, chunk=1)
        torch.cuda.synchronize()
        dev_ms, host_ms = [], []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(11):
            torch.cuda.synchronize()
            e0.record()
            det.focus_score(img_dev)
            e1.record()
            torch.cuda.synchronize()
            dev_ms.append(e0.elapsed_time(e1))
            t0 = time.perf_counter()
            s = det.focus_score_host(img_host, chunk=1)
            torch.cuda.synchronize()
            host_ms.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(dev_ms), statistics.median(host_ms), float(s[0])

    for name, size, bits, sig, n in (("C2", 1024, 8, (1.0, 10.0), 10), ("C3", 4096, 8, (1.0, 10.0), 10),
                                     ("C5", 8192, 16, (1.0, 30.0), 20)):
        img = synth.em_tile(size, size, 7 if name == "C5" else 1000, defocus=0.0, dose=300.0, bits=bits, device=dev)
        if bits == 16:   # as the C5 parity test: via numpy to a torch.uint16 tensor
            img = torch.from_numpy(img.to(torch.int32).cpu().numpy().astype(np.uint16)).to(dev)
        tau = 0.1 * (sig[1] - sig[0]) / n
        det = mhfd.Detector(size, size, sig[0], sig[1], n, threshold=tau, overlap=0.5, device=dev.index)
        dms, hms, score = timed(det, img.unsqueeze(0), img.unsqueeze(0).cpu().pin_memory())
        out[name] = {"size": size, "dtype": f"u{bits}", "sigma": list(sig), "scales": n, "schedule": det.schedule(
            f"u{bits}"), "device_ms": dms, "host_visible_ms": hms, "MPix_per_s_device": size * size / dms / 1e3,
            "score": score}
        if name in ("C2", "C3"):   # the same call replayed from a CUDA graph (launch gaps gone)
            out[name]["graph"] = graph_times(det, img.unsqueeze(0).contiguous(), score)
    out["C3_bands_1gpu"] = band_times(dev)
    out["C5_bands_1gpu"] = band_times(dev, c5=True)
    out["downsample_f2"] = downsample_times(dev)
    # C3 with the LoG response (reading R23): k_tc2 with 2n sub-levels
    # (row taps w / t^2 w2, column taps t^2 w2 / w, both column products into one accumulator)
    img = synth.em_tile(SIZE, SIZE, 1000, defocus=0.0, dose=300.0, device=dev)
    det = mhfd.Detector(SIZE, SIZE, SIGMA[0], SIGMA[1], NSCALES, threshold=0.1, overlap=OVERLAP,
                        device=dev.index, response="log")
    dms, hms, score = timed(det, img.unsqueeze(0), img.unsqueeze(0).cpu().pin_memory())
    fpp = det.schedule_flops_per_pixel("u8")
    out["C3_log"] = {"size": SIZE, "dtype": "u8", "sigma": list(SIGMA), "scales": NSCALES, "response": "log",
                     "schedule": det.schedule("u8"), "device_ms": dms, "host_visible_ms": hms,
                     "MPix_per_s_device": SIZE * SIZE / dms / 1e3, "score": score,
                     "tflops_issued": fpp * SIZE * SIZE / (dms * 1e-3) / 1e12,
                     "flop_kind": ("tensor fp16 split products (dense-equivalent band tiles)" if det.schedule("u8") == "k_tc2"
                                   else "fp32 direct convolutions")}
    # C3 in the 26-neighbour NMS mode (k_tc writes the DoG planes; k_nms26_roll) and with
    # the reflect boundary (k_tc with mirrored windows)
    for name, kw in (("C3_nms26", {"nms": "26"}), ("C3_reflect", {"boundary": "reflect"})):
        det = mhfd.Detector(SIZE, SIZE, SIGMA[0], SIGMA[1], NSCALES, threshold=TAU, overlap=OVERLAP,
                            device=dev.index, **kw)
        dms, hms, score = timed(det, img.unsqueeze(0), img.unsqueeze(0).cpu().pin_memory())
        out[name] = {"size": SIZE, "dtype": "u8", "sigma": list(SIGMA), "scales": NSCALES, **kw,
                     "schedule": det.schedule("u8"), "device_ms": dms, "host_visible_ms": hms,
                     "MPix_per_s_device": SIZE * SIZE / dms / 1e3, "score": score}
    return out


def graph_times(det, img, ref: float) -> dict:
    """One focus_score call captured in a CUDA graph (the call is stream-ordered with no
    host synchronisation, so it captures whole) and replayed: device time (CUDA events)
    and host-visible time (replay + synchronize), medians of 50."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        det.focus_score(img)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        out = det.focus_score(img)
    g.replay()
    torch.cuda.synchronize()
    assert float(out[0]) == ref, "graph replay score differs"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        g.replay()
    d, w = [], []
    for _ in range(50):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        w.append((time.perf_counter() - t0) * 1e3)
        d.append(e0.elapsed_time(e1))
    return {"device_ms": statistics.median(d), "host_visible_ms": statistics.median(w),
            "note": "device-resident image; torch.cuda.CUDAGraph replay of one mhfd_focus_score call"}


def downsample_times(dev) -> dict:
    """The bilinear downsampling pre-step (mhfd_downsample) on 16 x
    4096^2 u8 tiles (268 MB in, larger than L2) at factor 2: device time and achieved HBM
    bandwidth (bytes read + written) against the measured HBM peak."""
    import paper_2108_12050_b200 as mhfd
    B, f = 16, 2
    g = torch.Generator(device=dev).manual_seed(5)
    imgs = torch.randint(0, 256, (B, SIZE, SIZE), dtype=torch.uint8, device=dev, generator=g)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        mhfd.downsample(imgs, f)
    ms = []
    for _ in range(11):
        torch.cuda.synchronize()
        e0.record()
        mhfd.downsample(imgs, f)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = statistics.median(ms)
    nbytes = B * SIZE * SIZE * (1 + 1 / (f * f))
    pk, pk_note = peaks()
    return {"batch": B, "size": SIZE, "factor": f, "dtype": "u8", "device_ms": t, "GB_per_s": nbytes / t / 1e6,
            "hbm_peak_GB_per_s": pk.get("hbm_gbs"), "peak_note": pk_note,
            "hbm_frac": (nbytes / t / 1e6) / pk["hbm_gbs"] if pk.get("hbm_gbs") else None,
            "kernel": "k_downsample2<uint8_t>"}


def band_times(dev, c5: bool = False) -> dict:
    """Single-image sharding measured on one GPU: for G bands of one
    4096^2 u8 tile (k_tc) or, with c5, one 8192^2 u16 tile at sigma 1-30, 20 scales (the
    pair kernels), the device time of each rank's mhfd_detect_band (max over bands) and
    of mhfd_prune_candidates on the full list — the compute a G-GPU run does per image
    (the broadcast and the two all-gathers are not included)."""
    import synth
    import paper_2108_12050_b200 as mhfd
    from paper_2108_12050_b200.dist import band_rows, halo_rows
    size = 8192 if c5 else SIZE
    if c5:
        img = synth.em_tile(size, size, 7, defocus=0.0, dose=300.0, bits=16, device=dev)
        img = torch.from_numpy(img.to(torch.int32).cpu().numpy().astype(np.uint16)).to(dev)
        det = mhfd.Detector(size, size, 1.0, 30.0, 20, threshold=0.145, overlap=OVERLAP, device=dev.index)
    else:
        img = synth.em_tile(SIZE, SIZE, 1000, defocus=0.0, dose=300.0, device=dev)
        det = mhfd.Detector(SIZE, SIZE, SIGMA[0], SIGMA[1], NSCALES, threshold=TAU, overlap=OVERLAP,
                            device=dev.index)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def t(fn):
        for _ in range(3):
            fn()
        ms = []
        for _ in range(7):
            torch.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return statistics.median(ms)

    res = {"schedule": det.schedule("u16" if c5 else "u8")}
    for G in (1, 2, 4, 8):
        bands, parts = [], []
        for r in range(G):
            y0, y1 = band_rows(size, G, r)
            bands.append(t(lambda: det.detect_band(img, y0, y1)))
            c, nn = det.detect_band(img, y0, y1)
            parts.append(c[:int(nn)].clone())
        allc = torch.cat(parts, 0)
        pr = t(lambda: det.prune_candidates(allc, allc.shape[0]))
        # sharded pruning (mhfd_prune_band): each rank computes its band plus the halo
        # and prunes its own blobs; the ranks then only all-reduce three integers
        h = halo_rows(det)
        ext, certs = [], 0
        for r in range(G):
            y0, y1 = band_rows(size, G, r)
            a0, a1 = max(0, y0 - h), min(size, y1 + h)
            c, nn = det.detect_band(img, a0, a1)
            nn = int(nn)

            def band_and_prune():
                cc, n2 = det.detect_band(img, a0, a1)
                det.prune_band(cc, nn, a0, a1, y0, y1)
            ext.append(t(band_and_prune))
            certs += int(det.prune_band(c, nn, a0, a1, y0, y1)[1][0])
        res[str(G)] = {"band_ms_max": max(bands), "prune_ms": pr, "per_image_ms": max(bands) + pr,
                       "sharded_prune": {"halo_rows": h, "band_plus_prune_ms_max": max(ext), "certified": certs}}
    return res


def sharded_single_image(dev, dist, steps: int) -> dict:
    """Single-image sharding across the job's ranks (f2): one 4096^2 tile per step,
    broadcast + bands + all-gathers + pruning; device time, max over ranks."""
    import synth
    import paper_2108_12050_b200 as mhfd
    from paper_2108_12050_b200.dist import focus_score_single_image, focus_score_single_image_sharded
    img = synth.em_tile(SIZE, SIZE, 1000, defocus=0.0, dose=300.0, device=dev)
    det = mhfd.Detector(SIZE, SIZE, SIGMA[0], SIGMA[1], NSCALES, threshold=TAU, overlap=OVERLAP, device=dev.index)
    ref = float(det.focus_score(img)[0])
    for _ in range(3):
        focus_score_single_image(det, img)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        _, _, score, _ = focus_score_single_image(det, img)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    assert float(score[0]) == ref, "sharded score differs from the single-GPU score"
    # the same with the pruning sharded too (band + halo, certificate, one all-reduce)
    for _ in range(3):
        focus_score_single_image_sharded(det, img)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record()
    for _ in range(steps):
        _, score2, sharded = focus_score_single_image_sharded(det, img)
    e1.record()
    torch.cuda.synchronize()
    ms2 = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
    dist.all_reduce(ms2, op=dist.ReduceOp.MAX)
    assert score2 == ref, "sharded-pruning score differs from the single-GPU score"
    return {"workload": "one 4096^2 u8 tile per step, row bands across ranks (SURVEY §8(f) f2)",
            "ms_per_image": float(ms.item()), "score": ref,
            "sharded_pruning": {"ms_per_image": float(ms2.item()), "certified": bool(sharded)}}


# ------------------------------------------------------------------ GPU arm
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mhfd", choices=["mhfd", "reference"])
    ap.add_argument("--batch", type=int, default=64, help="images per GPU per step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C2/C3/C5 single-image measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.warmup < 3:
        log("warning: the contract asks for >= 3 warm-up steps")

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import paper_2108_12050_b200 as mhfd

    B = args.batch
    t0 = time.time()
    imgs = make_batch(rank, B, dev)
    torch.cuda.synchronize()
    log(f"[rank {rank}] generated {B} tiles in {time.time() - t0:.1f} s")
    det = mhfd.Detector(SIZE, SIZE, min_sigma=SIGMA[0], max_sigma=SIGMA[1], num_scales=NSCALES, threshold=TAU,
                        overlap=OVERLAP, device=local)
    from paper_2108_12050_b200.dist import gather_results
    gathered = torch.empty((world * B, 2), dtype=torch.float64, device=dev)

    def step():
        scores, counts = det.focus_score(imgs, counts=True)
        if dist is not None:   # the only collective: (count, score) of every image, 12 B each
            gather_results(counts, scores, gathered)
        return scores

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_call = mhfd.Detector.last_launch_count()

    det.timing_enable(args.steps)
    stream = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            scores = step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    stages = det.timing_read()
    det.timing_enable(0)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    px_step = world * B * SIZE * SIZE
    value = px_step / (ms_max * 1e-3) / 1e6

    # dominant kernel: the fused a2-a6 kernel (stage 1), averaged over the timed steps
    ss_ms = statistics.mean(s[1] for s in stages)
    stage_ms = {k: statistics.mean(s[i] for s in stages) for i, k in
                enumerate(["percentiles_a1", "blur_dog_argmax_a2_a6", "nms_compact_a7_a8", "prune_score_a9_a10"])}
    roofline = roofline_of(det, B, ss_ms, ms, stage_ms)

    # e2e through the host-buffer C-ABI entry point
    e2e = None
    if not args.no_e2e:
        host = imgs.cpu().pin_memory()
        for _ in range(2):
            det.focus_score_host(host, chunk=E2E_CHUNK)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        e0 = time.perf_counter()
        ev0.record(stream)
        for _ in range(args.steps):
            hs = det.focus_score_host(host, chunk=E2E_CHUNK)
            if dist is not None:
                gather_results(hs.to(dev), hs.to(dev), gathered)
        ev1.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - e0) * 1e3 / args.steps
        ems = torch.tensor([ev0.elapsed_time(ev1) / args.steps], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e_ms = float(ems.item())
        assert torch.equal(hs, scores.cpu()), "host-path scores differ from the device path"
        e2e = {"value": px_step / (e_ms * 1e-3) / 1e6, "unit": "MPix/s", "ms_per_step": e_ms,
               "wall_ms_per_step": wall, "h2d_bytes_per_step": B * SIZE * SIZE, "d2h_bytes_per_step": B * 12,
               "chunk": E2E_CHUNK,
               "api": "mhfd_focus_score_host (pinned host batch, three staging slots of E2E_CHUNK images, copies on a "
                      "second stream overlapped with compute; back-to-back steps pipeline, an idle device ramps "
                      "the chunks 1, 2, 3, ...)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(imgs[0].cpu().numpy())
    configs = None
    if rank == 0 and not args.no_configs:
        configs = other_configs(dev)
    sharded = None
    if dist is not None and not args.no_configs:
        try:   # an extra measurement: never let it take the main line down
            sharded = sharded_single_image(dev, dist, args.steps)
        except Exception as exc:  # noqa: BLE001
            sharded = {"error": repr(exc)[:300]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "MPix/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "ms_per_image": ms_max / B,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32 (k_tc: fp16 hi/lo split operands, f32 accumulation)",
                "data": "synthetic",
                "config": {"workload": "C4: per GPU a batch of 64 synthetic EM tiles 4096x4096 u8 (seed 1000+g, "
                                       "defocus 0.5*(g mod 9) px, dose 300); sigma 1-10, 10 scales, tau 0.09, "
                                       "overlap 0.5, Eq. 3 NMS",
                           "batch_per_gpu": B, "global_batch": world * B, "width": SIZE, "height": SIZE,
                           "parallelism": f"dp{world} (image sharding, NCCL all-gather of (count, score))",
                           "l2": "inputs larger than L2 (1.07 GB per GPU per step)"},
                "roofline": roofline, "stage_ms": stage_ms, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_call * args.steps, "clocks": clk.summary(), "other_configs": configs,
                "single_image_sharded": sharded,
                "mean_score": float(scores.mean())}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
