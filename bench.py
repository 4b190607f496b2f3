#!/usr/bin/env python
"""Bench of the PRNet pattern-attention forward on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload traffic] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

One step = one prnet_forward over the workload's whole test set (every
(window, channel) series), inputs resident in HBM.  Windows are sharded across
ranks (contiguous balanced ranges, no collective on the hot path); the only
collective is the all-reduce of the fp64 error sums (MSE/MAE) after the timed
region, plus the MAX of per-rank times.  Rank 0 prints ONE JSON line.

--impl reference times the CPU oracle (oracle/, as it stands) on the host
cores on a bounded sample of the same workload -- this tier's reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "PRNet forward windows/sec and HBM GB/s vs peak at 1/2/4/8 B200"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


def flops_per_series(N, S, M):
    """Algorithmic FLOPs of the folded formulation: Gram 2N^2S,
    fold Q = W_s A_s + W_t A_t 4MN^2, Y = Q X 2MNS."""
    return 2 * N * N * S + 4 * M * N * N + 2 * M * N * S


def _up(v, m):
    return -(-v // m) * m


def tensor_flops_per_series(variant, N, S, M):
    """FLOPs the tensor cores are ISSUED per series by a tensor-core variant (split-fp16 hi/lo:
    3 products per contraction, tiles padded to the MMA shapes), or None for the CUDA-core
    FP32 variants.  tc_quad: Gram of a quad on tcgen05 (M = N = 128, 5 K-steps of 16; 4x of
    it is the discarded off-diagonal blocks), fold on tcgen05 (12 MMAs M = 128, N = 32,
    K = 16 per quad), head on mma.sync (36 m16n8k16 per series).  mma_f16x3 / flash_f16x3:
    m16n8k16 tiles of the Gram, of the fold (mma) or of P = E X (flash), and of the head."""
    NP, MP, SP, KZ = _up(N, 16), _up(M, 16), _up(S, 8), _up(S, 16)
    if variant == "tc_quad" and S == 24:   # M <= 16: fold N = 16 and one head m-tile (MTL = 1)
        mf, mt = (16, 1) if M <= 16 else (32, 2)
        return (5 * 2 * 128 * 128 * 16 + 12 * 2 * 128 * mf * 16) / 4 + 18 * mt * 2 * 16 * 8 * 16
    if variant == "tc_quad":   # generic S (fwd_tcg.cu): 3 runs of KZ/16 Gram K-steps, fold N 16/32/64
        mf = 16 if M <= 16 else (32 if M <= 32 else 64)
        return ((3 * (KZ // 16) * 2 * 128 * 128 * 16 + 12 * 2 * 128 * mf * 16) / 4
                + 3 * (MP // 16) * (SP // 8) * 2 * 2 * 16 * 8 * 16)
    if variant == "tc_long":   # fwd_tcl.cu: 128-row query x 64-key tiles, Gram + P = E X' + head
        nqt, nkt = -(-N // 128), -(-N // 64)
        nm = 2 if 320 + 4 * KZ <= 512 else 1
        gram = 3 * (KZ // 16) * 2 * 128 * 64 * 16
        pmma = (16 * 2 * 128 * 2 * KZ * 16) if nm == 2 else (24 * 2 * 128 * KZ * 16)
        head = nqt * 4 * 2 * (SP // 8) * 2 * (MP // 16) * 3 * 2 * 16 * 8 * 16
        return nqt * nkt * (gram + pmma) + head
    if variant == "mma_f16x3":
        return 3 * 2 * (NP * NP * KZ + 2 * MP * NP * NP + MP * SP * NP)
    if variant == "flash_f16x3":
        return 3 * 2 * (NP * NP * KZ + 2 * NP * NP * SP + 2 * MP * NP * SP)
    return None


# inputs up to this size get an L2 flush between timed steps (B200 L2: 126 MB)
L2_FLUSH_BELOW = 256 << 20

# ------------------------------------------------------------------ clocks (NVML, sampled in a thread)
class ClockSampler:
    BAD = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
           "hw_power_brake": 0x80}
    ALL = {"gpu_idle": 0x1, "applications_clocks": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
           "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
           "hw_power_brake": 0x80, "display_clocks": 0x100}

    def __init__(self, device_index, period_s=0.005):
        self.samples, self.reasons, self.power = [], 0, []
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
        self.period = period_s

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.power.append(nv.nvmlDeviceGetPowerUsage(self._h) / 1000.0)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        reasons = [k for k, v in self.ALL.items() if self.reasons & v]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples),
                "power_w_median": statistics.median(self.power) if self.power else None}


# ------------------------------------------------------------------ CPU oracle leg
_ORACLE_CACHE = {}


def _oracle_chunk(args):
    """Worker: oracle.forward (as it stands, 1 thread) on whole windows of a channel block."""
    name, seed, widx, chans = args
    import oracle
    key = (name, seed, tuple(widx), tuple(chans))
    if key not in _ORACLE_CACHE:
        w = synth.WORKLOADS[name]
        N, _, M = synth.derived_dims(w.L, w.S, w.H)
        s = synth.make_series(w, seed, channels=chans)
        x, _ = synth.window_batch(s, w, widx)
        ws, wt, b = synth.make_params(w.C, M, N, w.H, True, seed, w.cfg_id)
        _ORACLE_CACHE.clear()
        _ORACLE_CACHE[key] = (x, ws[chans], wt[chans], b[chans], w.S, w.H)
    x, ws, wt, b, S, H = _ORACLE_CACHE[key]
    t0 = time.perf_counter()
    oracle.forward(x, S, H, ws, wt, b, True)
    return time.perf_counter() - t0, x.shape[0] * x.shape[1]


class CpuOracleBench:
    """The oracle timed on the host cores on a bounded, fixed sample of the workload:
    whole windows (all channels) spread evenly over the test set, split by channel
    blocks over one single-threaded process per core.  step() returns windows/s."""

    def __init__(self, name, seed, budget_s=3.0, cores=None):
        import multiprocessing as mp
        import oracle
        oracle.build()
        self.w = w = synth.WORKLOADS[name]
        self.cores = cores or len(os.sched_getaffinity(0))
        dt, n = _oracle_chunk((name, seed, [0], list(range(min(w.C, 8)))))
        per_series = dt / n
        n_series = max(w.C, int(budget_s * self.cores / per_series))
        n_win = max(1, min(w.windows, n_series // w.C))
        self.widx = np.unique(np.linspace(0, w.windows - 1, n_win).astype(int)).tolist()
        blocks = [b.tolist() for b in np.array_split(np.arange(w.C), min(self.cores, w.C)) if len(b)]
        self.jobs = [(name, seed, self.widx, blk) for blk in blocks]
        self.pool = mp.get_context("fork").Pool(len(self.jobs))
        self.pool.map(_oracle_chunk, self.jobs)          # build the inputs in the workers

    def step(self):
        t0 = time.perf_counter()
        res = self.pool.map(_oracle_chunk, self.jobs)
        self.wall = time.perf_counter() - t0
        self.compute = max(r[0] for r in res)
        self.series = sum(r[1] for r in res)
        return self.series / self.compute / self.w.C

    def describe(self):
        w = self.w
        return (f"{len(self.widx)} of {w.windows} windows x {w.C} channels ({self.series} series) "
                f"per step, {len(self.jobs)} processes x 1 thread, {self.compute:.2f} s compute "
                f"(wall {self.wall:.2f} s)")

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_oracle_rate(name, seed, budget_s=12.0, cores=None):
    """One timed pass of the oracle over a ~budget_s sample: (windows/s, series/s, cores, sample)."""
    b = CpuOracleBench(name, seed, budget_s, cores)
    wps = b.step()
    desc = b.describe()
    b.close()
    return wps, wps * b.w.C, len(b.jobs), desc


# ------------------------------------------------------------------ distributed helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="traffic", choices=sorted(synth.WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=synth.DEFAULT_SEED)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu (no extras)")
    ap.add_argument("--variant", default=None, help="force a kernel variant (tuning)")
    ap.add_argument("--metric-variant", type=int, default=0,
                    help="SURVEY 8(f) f3: bit 0 level-only trend, bit 1 detrended seasonal, "
                         "bit 2 component values")
    ap.add_argument("--graph", action="store_true",
                    help="time replays of a CUDA graph of the forward call (launch-bound configs)")
    ap.add_argument("--ma-kernel", type=int, default=0,
                    help="SURVEY 8(f) f3: moving-average decomposition kernel (odd, 0 = off)")
    ap.add_argument("--instance-norm", action="store_true",
                    help="SURVEY 8(f) f1: RevIN-style instance normalisation")
    ap.add_argument("--sliding", action="store_true",
                    help="SURVEY 8(f) f2: forecast the test windows straight from the [C][T] "
                         "series (prnet_forward_sliding); e2e uploads the series span once")
    ap.add_argument("--host-chunk", type=int, default=0,
                    help="windows per chunk of the host-buffer pipeline (0 = library default)")
    args = ap.parse_args()

    rank, world, local = dist_env()
    w = synth.WORKLOADS[args.workload]
    N, r, M = synth.derived_dims(w.L, w.S, w.H)
    B = w.windows
    cfg = {"workload": w.name, "windows": B, "C": w.C, "L": w.L, "S": w.S, "H": w.H, "N": N,
           "M": M, "series_per_step": B * w.C, "head": "per-channel",
           "l2": (f"inputs larger than L2 ({B * w.C * w.L * 4 / 1e9:.2f} GB read per step)"
                  if B * w.C * w.L * 4 > L2_FLUSH_BELOW else
                  f"L2 flushed between timed steps (512 MB write; inputs {B * w.C * w.L * 4 / 1e6:.1f}"
                  f" MB < L2)"),
           "parallelism": f"dp{world}", "seed": args.seed}
    if args.metric_variant or args.instance_norm or args.ma_kernel:
        cfg.update(metric_variant=args.metric_variant, instance_norm=bool(args.instance_norm),
                   ma_kernel=args.ma_kernel)
    if args.sliding:
        cfg.update(input="sliding windows of the [C][T] series (prnet_forward_sliding)",
                   l2=f"series span {w.C * (B + w.L - 1) * 4 / 1e6:.1f} MB < L2: L2 flushed "
                      f"between timed steps (512 MB write); outputs "
                      f"{B * w.C * w.H * 4 / 1e9:.2f} GB written per step")

    if args.impl == "reference":
        if rank != 0:
            return 0
        # each step: one oracle pass over a fixed sample sized so the whole run takes minutes
        per_step = max(0.3, min(3.0, 150.0 / max(1, args.steps + args.warmup)))
        ob = CpuOracleBench(w.name, args.seed, budget_s=per_step)
        for _ in range(args.warmup):
            ob.step()
        rates, sample_s = [], []
        for _ in range(args.steps):
            rates.append(ob.step())
            sample_s.append(ob.compute)
        value = len(rates) / sum(1.0 / r for r in rates)      # windows / total time
        sample = ob.describe()
        cores = len(ob.jobs)
        ob.close()
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": value, "unit": "windows/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * B / value, "higher_is_better": True, "scaling": "strong",
            "ms_per_step_note": ("EXTRAPOLATED to the whole workload from the measured sample "
                                 "rate; each timed step runs only the sample "
                                 "(sample_ms_per_step, measured)"),
            "sample_ms_per_step": 1e3 * statistics.mean(sample_s),
            "sample_windows_per_step": len(ob.widx),
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": "windows/s", "cores": cores,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "windows/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return 0

    import torch
    import torch.distributed as dist
    from paper_2404_02445_b200 import PRNet, all_reduce_error_sums, shard_windows

    # one process per GPU; NCCL for the collectives.  (world > GPUs only happens in the
    # single-GPU multi-rank smoke test: ranks then share a device and collectives use gloo
    # on host tensors -- a functional check of the sharding/reduction path, not a timing.)
    ndev = torch.cuda.device_count()
    dev = local % ndev
    torch.cuda.set_device(dev)
    use_nccl = world > 1 and ndev >= world
    if world > 1:
        if use_nccl:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    coll = "cuda" if (use_nccl or world == 1) else "cpu"
    cfg["collectives"] = "nccl" if use_nccl else ("gloo (shared-GPU smoke test)" if world > 1 else "none")
    start, count = shard_windows(B, world, rank)
    peaks, peak_src = measured_peaks()

    # ---- inputs: this rank's windows, materialised in HBM (outside the timed region)
    series = synth.make_series(w, args.seed)
    sd = torch.from_numpy(series).cuda()
    x = sd.unfold(1, w.L, 1)[:, w.t0 + start:w.t0 + start + count, :].permute(1, 0, 2).contiguous()
    tgt = sd[:, w.L:].unfold(1, w.H, 1)[:, w.t0 + start:w.t0 + start + count, :] \
        .permute(1, 0, 2).contiguous()
    if not args.sliding:
        del sd
    ws, wt, b = synth.make_params(w.C, M, N, w.H, True, args.seed, w.cfg_id)
    model = PRNet(w.C, w.L, w.S, w.H, device=dev, metric_variant=args.metric_variant,
                  instance_norm=args.instance_norm, ma_kernel=args.ma_kernel).load(ws, wt, b)
    if args.variant:
        model.set_variant(args.variant)
    y = torch.empty((count, w.C, w.H), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    plan = model.plan(count)

    if args.sliding:
        t0s = w.t0 + start
        y_ref = model.forward(x)
        del x
        fwd = lambda: model.forward_sliding_into(sd, t0s, count, y, stream)  # noqa: E731
        fwd()
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref), "sliding forward disagrees with the materialised windows"
        del y_ref
    else:
        fwd = lambda: model.forward_into(x, y, stream)  # noqa: E731
    for _ in range(args.warmup):
        fwd()
    torch.cuda.synchronize()
    if args.graph and not args.sliding:
        # launch-bound workloads (configs[0]): the step is one replay of a captured CUDA graph
        # of the same prnet_forward call, so host launch overhead leaves the timed region
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            model.forward_into(x, y)
        graph.replay()
        torch.cuda.synchronize()
        fwd = graph.replay
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    # inputs smaller than L2 (126 MB): flush it between timed steps (outside the brackets) and
    # time the steps by their own event pairs
    flush = None
    if count * w.C * w.L * 4 <= L2_FLUSH_BELOW or args.sliding:
        flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)   # 512 MB
    nvtx = torch.cuda.nvtx
    with ClockSampler(dev) as clk:
        t_wall = time.perf_counter()
        nvtx.range_push(f"bench timed region: {args.steps} steps of {w.name}")
        for k, (e0, e1) in enumerate(ev):
            if flush is not None:
                nvtx.range_push("L2 flush (untimed)")
                flush.zero_()
                nvtx.range_pop()
            nvtx.range_push(f"step {k}: prnet_forward ({count} windows x {w.C} channels)")
            e0.record(stream)
            fwd()
            e1.record(stream)
            nvtx.range_pop()
        nvtx.range_pop()
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    per_launch = [e0.elapsed_time(e1) for e0, e1 in ev]          # ms, on the launching stream
    total_ms = ev[0][0].elapsed_time(ev[-1][1]) if flush is None else sum(per_launch)
    tt = torch.tensor([total_ms], dtype=torch.float64, device=coll)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total_ms_max = float(tt.item())
    ms_per_step = total_ms_max / args.steps

    # ---- accuracy metric of this forward (K6 error sums + the one NCCL all-reduce)
    sums = model.error_sums(y, tgt).to(coll)
    mse, mae = all_reduce_error_sums(sums)

    if args.profile:
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_per_step}), flush=True)
        return 0

    # ---- end to end through the public API with HOST buffers (H2D + kernel + D2H timed)
    e2e = None
    if not args.no_e2e and args.sliding:
        try:
            sh = torch.empty(sd.shape, dtype=torch.float32, pin_memory=True)
            sh.copy_(sd)
            yh = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
            model.forward_sliding_host(sh, t0s, count, yh,
                                       chunk_windows=args.host_chunk or None)   # warm-up
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                model.forward_sliding_host(sh, t0s, count, yh)
            dt = torch.tensor([(time.perf_counter() - t0) / args.e2e_steps], dtype=torch.float64,
                              device=coll)
            if world > 1:
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            assert torch.equal(yh, y.cpu()), "host sliding path disagrees with the device path"
            e2e = {"value": B / float(dt.item()), "unit": "windows/s",
                   "h2d_bytes_per_step": int(w.C * (count + w.L - 1) * 4) * world,
                   "d2h_bytes_per_step": int(yh.numel() * 4) * world,
                   "steps": args.e2e_steps,
                   "path": "prnet_forward_sliding_host (pinned host series, span uploaded once)"}
            del sh, yh
        except Exception as ex:  # report, never fake
            e2e = {"value": None, "unit": "windows/s", "error": str(ex)[:200]}
    elif not args.no_e2e:
        try:
            xh = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
            xh.copy_(x)
            yh = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
            model.forward_host(xh, yh, chunk_windows=args.host_chunk or None)   # warm-up
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                model.forward_host(xh, yh)
            dt = torch.tensor([(time.perf_counter() - t0) / args.e2e_steps], dtype=torch.float64,
                              device=coll)
            if world > 1:
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            assert torch.equal(yh, y.cpu()), "host path disagrees with the device path"
            e2e = {"value": B / float(dt.item()), "unit": "windows/s",
                   "h2d_bytes_per_step": int(xh.numel() * 4) * world,
                   "d2h_bytes_per_step": int(yh.numel() * 4) * world,
                   "steps": args.e2e_steps, "path": "prnet_forward_host (pinned host buffers)"}
            del xh, yh
        except Exception as ex:  # report, never fake
            e2e = {"value": None, "unit": "windows/s", "error": str(ex)[:200]}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    value = B / (ms_per_step / 1e3)
    bytes_per_series = 4 * (w.L + w.H)
    launch_bytes = count * w.C * bytes_per_series
    if args.sliding:   # the series span is read once, the outputs written once
        bytes_per_series = 4 * w.H + 4 * (count + w.L - 1) / count
        launch_bytes = 4 * w.C * (count + w.L - 1) + 4 * count * w.C * w.H
    launch_ms = statistics.mean(per_launch)
    achieved_gbs = launch_bytes / (launch_ms / 1e3) / 1e9
    peak_gbs = float(peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"]))
    fl = flops_per_series(N, w.S, M)
    achieved_tf = count * w.C * fl / (launch_ms / 1e3) / 1e12
    clocks = clk.summary()
    sm_clock = (clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            # measured for one full-workload launch of the plain path: scaled to this rank's
            # share of the windows; not applicable to the sliding or widened modes
            t_full = json.load(open(prof)).get(w.name)
            widened = args.sliding or args.metric_variant or args.instance_norm or args.ma_kernel
            traffic = None if (widened or t_full is None) else t_full * count / w.windows
        except Exception:
            traffic = None
    traffic_src = ("STATIC: dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full "
                   "capture of this workload's launch (profiles/ncu_traffic.json, tools/"
                   "summarize_profile.py), scaled to this rank's windows; not measured in this run"
                   if traffic is not None else "no ncu capture for this mode")
    tflops = tensor_flops_per_series(plan["variant"], N, w.S, M)

    cpu = None
    if world == 1 and not args.no_cpu_baseline and not (args.metric_variant or args.instance_norm
                                                        or args.ma_kernel):
        try:
            wps, sps, cores, sample = cpu_oracle_rate(w.name, args.seed, args.cpu_budget)
            cpu = {"value": wps, "unit": "windows/s", "cores": cores, "kind": "oracle",
                   "sample": sample, "series_per_s": sps}
        except Exception as ex:
            cpu = {"value": None, "unit": "windows/s", "error": str(ex)[:200]}

    out = {
        "metric": METRIC, "value": value, "unit": "windows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seasonal+trend+noise series, random-init head; DESIGN.md §5)",
        "config": cfg,
        "series_per_s": value * w.C,
        "hbm_gbs": B * w.C * bytes_per_series / (ms_per_step / 1e3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": peak_gbs, "unit": "GB/s",
                     "frac": achieved_gbs / peak_gbs, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "kernel": f"prnet_fwd_{plan['variant']}", "launch_ms": launch_ms,
                     "bytes_per_launch": launch_bytes, "peak_source": peak_src},
        "roofline_compute": (
            {"bound": "tensor", "unit": "TFLOP/s",
             "achieved": count * w.C * tflops / (launch_ms / 1e3) / 1e12,
             "peak": float(peaks.get("bf16_tflops_sustained", 1400.0)),
             "frac": count * w.C * tflops / (launch_ms / 1e3) / 1e12
             / float(peaks.get("bf16_tflops_sustained", 1400.0)),
             "issued_flops_per_series": tflops, "algorithmic_flops_per_series": fl,
             "peak_source": f"{peak_src}: bf16_tflops_sustained (f16 dense = bf16 rate)",
             "note": "ISSUED tensor FLOPs: split-fp16 3 products, tile padding, tc_quad's "
                     "block-diagonal Gram waste; the mma.sync share runs at ~1/4 of the "
                     "tcgen05 peak (profiles/r01_microbench.txt: 554 TF/s)"}
            if tflops is not None else
            {"bound": "alu", "achieved": achieved_tf, "unit": "TFLOP/s",
             "peak": fp32_peak, "frac": achieved_tf / fp32_peak,
             "flops_per_series": fl,
             "peak_note": "FP32 FFMA: 148 SMs x 128 lanes x 2 x max SM clock (CUDA-core variant)"}),
        "accuracy": {"mse": mse, "mae": mae},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": plan["kernel_launches"] * args.steps,
        "clocks": clocks,
        "wall_s_timed_region": t_wall,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
