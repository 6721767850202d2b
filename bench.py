#!/usr/bin/env python
"""Benchmark: denoised images/s for the full Noise2Fast fit-and-denoise of a
512x512 image (BASELINE.json configs[1]) on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one complete fit-and-denoise of one image (normalise, pairs,
init, every epoch until the early stop, window mean) with the reference's
default TrainConfig.  N > 1 runs under torchrun, one process per GPU, each
rank fitting its own images (no collective on the data path: weak scaling).

ours:       value = images/s with the input resident in HBM (Engine.fit_device,
            CUDA events on the engine stream, max over ranks); e2e = the same
            metric through the public API train_single_channel() with the
            input in pinned host memory (H2D + D2H inside the timed region).
reference:  the CPU oracle port (oracle/n2f_oracle.py) on the host cores, one
            training epoch per step, extrapolated to a full fit with the
            epoch count of the GPU fit of the same image (see --ref-epochs).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "denoised images/sec (512x512 gray) at 1/2/4/8 B200; conv tensor-pipe % of peak"
UNIT = "images/s"
SIZE = 512
SEED = 0
EPOCHS_FILE = os.path.join(ROOT, "profiles", "bench_epochs.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--conv-impl", type=int, default=0)
    p.add_argument("--ref-epochs", type=int, default=None,
                   help="epochs of a full fit used to extrapolate the CPU per-epoch time")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--host-loop", action="store_true",
                   help="launch every kernel from the host instead of the captured while-graph "
                        "(the same kernels; for ncu launch lists, which cannot see kernels inside "
                        "conditional graph nodes)")
    p.add_argument("--workload", choices=["config2", "batch64"], default="config2",
                   help="config2: K fits of the 512x512 image per GPU (weak scaling); batch64: "
                        "BASELINE config 4, 64 images shared by all GPUs through a dynamic "
                        "queue (strong scaling)")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def workload():
    from paper_2108_10209_b200 import synthetic

    noisy, clean = synthetic.config_image(2, SEED)  # 512x512, sigma 50/255, seeded
    return noisy, clean


def config_block(n_gpus):
    return {"workload": "config2: one 512x512 blob+rect image, gaussian sigma=50/255, seed 0; full "
                        "fit-and-denoise, reference default TrainConfig (bce, checkerboard, lr 1e-3, "
                        "patience 100, window 100)",
            "image": [SIZE, SIZE], "images_per_step_per_gpu": 1,
            "parallelism": f"independent images, {n_gpus} GPU(s), no collective",
            "l2": "working set (activations ~1.5 GB) exceeds the 126 MB L2; no flush needed"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["bf16_tflops"]), float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 6650.0, "fallback"


def load_sustained_tflops():
    """cuBLAS bf16 back to back for 4 s (MEASURED_PEAKS.json), or None."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops_sustained"])
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for n, v in zip(names, r[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU legs (oracle port) -- only here may bench.py execute oracle/
# ---------------------------------------------------------------------------


def cpu_epoch_seconds(noisy: np.ndarray, reps: int = 1) -> tuple[float, int]:
    """Time one training epoch (4 Adam steps + full-res validation) of the
    oracle on the host cores; returns (seconds per epoch, BLAS threads)."""
    from oracle import n2f_oracle as o

    try:
        from threadpoolctl import threadpool_info

        threads = max([d.get("num_threads", 1) for d in threadpool_info()
                       if d.get("user_api") == "blas"] or [1])
    except Exception:
        threads = os.cpu_count() or 1
    norm, lo, hi, _ = o.normalize(noisy)
    n32 = norm.astype(np.float32)
    pairs = o.training_pairs(n32)
    net = o.init_net(SEED)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for a, b in pairs:
            z, cache = o.net_forward(net, a, keep=True)
            _, gz = o.bce_logits(z, b)
            o.net_step(net, o.net_backward(net, cache, gz), 1e-3)
        out = o.predict(net, n32)
        o.val_score(out, n32)
        times.append(time.perf_counter() - t0)
    return min(times), threads


def recorded_epochs(default=None):
    try:
        with open(EPOCHS_FILE) as f:
            return int(json.load(f)["epochs_run"])
    except Exception:
        return default


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    noisy, _ = workload()
    epochs = args.ref_epochs or recorded_epochs(150)
    for _ in range(max(0, min(args.warmup, 1))):  # one warm-up epoch primes BLAS/allocations
        cpu_epoch_seconds(noisy)
    t0 = time.perf_counter()
    per = []
    threads = 1
    for _ in range(args.steps):
        s, threads = cpu_epoch_seconds(noisy)
        per.append(s)
    wall = time.perf_counter() - t0
    s_epoch = sum(per) / len(per)
    value = 1.0 / (s_epoch * epochs)
    sample = (f"one training epoch (4 Adam steps + 512x512 validation) of the oracle port per step, "
              f"{s_epoch:.2f} s/epoch, extrapolated x{epochs} epochs (epochs_run of the GPU fit of the "
              f"same image)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * s_epoch * epochs, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_block(world), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def run_ours(args):
    import torch

    from paper_2108_10209_b200 import Engine, TrainConfig, _lib, train_single_channel
    from paper_2108_10209_b200 import trainer as T

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    os.environ["N2F_DEVICE"] = str(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    noisy, clean = workload()
    cfg = TrainConfig(seed=SEED)
    eng = Engine(SIZE, SIZE, cfg, device=local, conv_impl=args.conv_impl, use_graph=not args.host_loop)
    stream = torch.cuda.ExternalStream(eng.stream)
    img = torch.from_numpy(noisy).cuda()
    out = torch.empty((SIZE, SIZE), dtype=torch.float64, device="cuda")

    def fit():
        return eng.fit_device(img.data_ptr(), _lib.N2F_F32, out.data_ptr())

    for _ in range(args.warmup):
        r = fit()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    epochs = []
    e0.record(stream)
    for _ in range(args.steps):
        r = fit()
        launches += r.kernel_launches
        epochs.append(r.epochs_run)
    e1.record(stream)
    e1.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * args.steps / (max_ms / 1e3)
    denoised = out.cpu().numpy()

    # ---- e2e through the public API, input in pinned host memory ----------
    pinned = torch.empty((SIZE, SIZE), dtype=torch.float32).pin_memory()
    pinned.copy_(torch.from_numpy(noisy))
    host_in = pinned.numpy()
    res = train_single_channel(host_in, cfg)  # builds / warms the cached engine
    api_eng = next(iter(T._cache.values()))
    api_stream = torch.cuda.ExternalStream(api_eng.stream)
    barrier()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(api_stream)
    for _ in range(args.steps):
        res = train_single_channel(host_in, cfg)
    a1.record(api_stream)
    a1.synchronize()
    t2 = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_value = world * args.steps / (float(t2.item()) / 1e3)
    h2d = SIZE * SIZE * 4
    d2h = SIZE * SIZE * 8 + res.epochs_run * (8 + 32 + 8) + 64

    # ---- dominant kernel roofline: one profiled epoch on the same engine and
    # stream right after the timed region (CUDA events around every launch)
    peak_tf, peak_gbs, peak_kind = load_peaks()
    pms, pfl, pln = eng.profile_epoch()
    ci, li = np.unravel_index(int(np.argmax(pms)), pms.shape)
    kms = float(pms[ci, li] / max(1, pln[ci, li]))
    kflop = float(pfl[ci, li] / max(1, pln[ci, li]))
    achieved = kflop / (kms * 1e-3) / 1e12
    kname = f"{Engine.PROF_CLASSES[ci]} layer {li + 1} ({pln[ci, li]} launches/epoch)"
    shares = {name: round(float(pms[i].sum() / pms.sum()), 4) for i, name in enumerate(Engine.PROF_CLASSES)}
    epoch_ms_profiled = float(pms.sum())
    conv_tf = float(pfl[[1, 3, 4, 8]].sum() / (pms[[1, 3, 4, 8]].sum() * 1e-3) / 1e12)
    # the split-precision kernels issue 3 MMAs per algorithmic MAC: FP16x3 at
    # the fp16/bf16 dense rate (the default), 3xTF32 at half that rate
    if args.conv_impl == 2:
        mma_note, mma_cost = "3xTF32: 3 tf32 MMAs (half the bf16 rate) per algorithmic MAC", 2.0
    elif args.conv_impl == 1:
        mma_note, mma_cost = "SIMT fp32 (no tensor cores)", 0.0
    else:
        mma_note, mma_cost = "FP16x3: 3 fp16 MMAs (bf16 dense rate) per algorithmic MAC", 1.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "dominant_kernel_traffic.json")) as f:
            tj = json.load(f)
        # only when the capture is of the kernel this run found dominant
        if kname.startswith(tj.get("kernel", "?")):
            traffic = tj.get("dram_bytes_per_launch")
    except Exception:
        pass

    if rank == 0:
        os.makedirs(os.path.dirname(EPOCHS_FILE), exist_ok=True)
        try:
            with open(EPOCHS_FILE, "w") as f:
                json.dump({"epochs_run": int(epochs[-1]), "config": "config2 seed 0"}, f)
        except Exception:
            pass
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        s_epoch, threads = cpu_epoch_seconds(noisy)
        cpu_value = 1.0 / (s_epoch * epochs[-1])
        cpu = {"value": cpu_value, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"one training epoch (4 Adam steps + 512x512 validation) of the oracle port, "
                         f"{s_epoch:.2f} s, extrapolated x{epochs[-1]} epochs (this GPU fit's epochs_run)"}
    psnr_in = 10 * np.log10(1.0 / np.mean((noisy.astype(np.float64) - clean) ** 2))
    psnr_out = 10 * np.log10(1.0 / np.mean((denoised - clean) ** 2))
    epoch_flop = 16392512.0 * SIZE * SIZE
    path_tflops = epoch_flop * epochs[-1] * world * args.steps / (max_ms * 1e-3) / 1e12
    sus_tf = load_sustained_tflops()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_block(world),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "traffic": traffic,
                         "kernel": kname, "kernel_ms": kms, "kernel_algorithmic_flop": kflop,
                         "peak_kind": f"{peak_kind} bf16 dense burst; {mma_note}",
                         "mma_frac": achieved * 3 * mma_cost / peak_tf,
                         "conv_kernels_tflops": conv_tf, "epoch_ms_profiled": epoch_ms_profiled,
                         "time_share": shares,
                         "path_tflops": path_tflops, "path_frac": path_tflops / peak_tf,
                         # the whole timed fit against the sustained tensor rate (cuBLAS bf16
                         # back to back, MEASURED_PEAKS.json), with the 3 MMAs per MAC counted
                         "peak_sustained": sus_tf,
                         "path_mma_frac_sustained": (path_tflops * 3 * mma_cost / sus_tf) if sus_tf else None},
            "cpu_baseline": cpu,
            "clocks": clk,
            "epochs_run": epochs, "psnr_noisy_db": psnr_in, "psnr_denoised_db": psnr_out,
            # the stable kernel-side number: the early-stop epoch count of one
            # image moves with last-bit changes (chaotic training)
            "ms_per_epoch": max_ms / args.steps / epochs[-1],
        }
        print(json.dumps(line), flush=True)
    eng.close()
    T.release_engines()
    if dist is not None:
        dist.destroy_process_group()


def run_batch64(args):
    """BASELINE config 4: 64 independent 512x512 images (per-image seed, sigma
    ~ U(15,50)/255) shared by all ranks through a store-backed dynamic queue;
    value = 64 / max-over-ranks device time (strong scaling)."""
    import torch

    from paper_2108_10209_b200 import Engine, TrainConfig, _lib, pool, synthetic

    rank, local, world = pool.dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_img = 64
    images = [synthetic.config_image(4, seed=1000 + i)[0] for i in range(n_img)]
    eng = Engine(SIZE, SIZE, TrainConfig(seed=0), device=local, conv_impl=args.conv_impl,
                 use_graph=not args.host_loop)
    stream = torch.cuda.ExternalStream(eng.stream)
    out = torch.empty((SIZE, SIZE), dtype=torch.float64, device="cuda")
    img = torch.empty((SIZE, SIZE), dtype=torch.float32, device="cuda")
    for _ in range(max(1, args.warmup)):  # warm the engine (graph, caches) on image 0
        img.copy_(torch.from_numpy(images[0]))
        eng.fit_device(img.data_ptr(), _lib.N2F_F32, out.data_ptr())
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    store = pool.default_store()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    done, epochs = [], []
    for i in pool.claim(store, "bench/batch64", n_img):
        img.copy_(torch.from_numpy(images[i]), non_blocking=False)
        eng.set_seed(1000 + i)  # per-image network seed, like the CLI's per-file seeds
        r = eng.fit_device(img.data_ptr(), _lib.N2F_F32, out.data_ptr())
        done.append(i)
        epochs.append(r.epochs_run)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    max_ms = pool.max_over_ranks(ms, device="cuda")
    total_epochs = pool.sum_over_ranks(sum(epochs), device="cuda")
    busy_ms = pool.gather_over_ranks(ms, device="cuda")
    n_per_rank = pool.gather_over_ranks(len(done), device="cuda")
    flop = 16_392_512.0 * SIZE * SIZE * total_epochs  # FLOP per pixel-epoch
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": n_img / (max_ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": 1, "warmup": args.warmup, "ms_per_step": max_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "config4: 64 independent 512x512 blob+rect images, per-image "
                                   "seed, gaussian sigma ~ U(15,50)/255, dynamic queue over GPUs",
                       "images": n_img, "parallelism": f"{world} GPU(s), no collective on the data path"},
            "rank0_images": len(done), "rank0_ms": ms, "total_epochs": total_epochs,
            "per_gpu_busy_ms": busy_ms, "per_gpu_images": n_per_rank,
            "imbalance_max_over_mean": pool.imbalance(busy_ms),
            "algorithmic_tflops_per_gpu": flop / (max_ms * 1e-3) / world / 1e12,
        }), flush=True)
    eng.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "batch64":
        run_batch64(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
