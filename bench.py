"""Benchmark: video tokens/s per denoise step of the Vchitect-2.0 2B block (bf16).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config 2]

One "step" = one parallel MM-DiT block forward (model.py:263-271) over the
config's synthetic clip. N=1: BASELINE.json configs[1] (config 2: 16 frames x
30x45 patches + 256 text tokens, D 1584, H 24, bf16) on one B200, inputs
resident in HBM. N>1 (torchrun, one rank per GPU, NCCL): the same block
sequence-parallel (spatial shard axis, head-parallel all-to-all), strong
scaling, time = max over ranks.

Rank 0 prints ONE JSON line (contract in the task statement). Extra keys:
roofline (dominant kernel, from the library's per-stage CUDA-event profiler
in a separate untimed pass), cpu_baseline (the oracle port on this host's
cores, bounded sample), e2e (C-ABI call with pinned HOST buffers: H2D of the
inputs and D2H of the block output inside the timed region), clocks.

--impl reference times the reference algorithm's CPU implementation (the
pinned oracle port, oracle/spsim_oracle.py; the reference is pure Python and
cannot travel to the GPU box) on the same config, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # id: (F, Lv, Lt, D, H, name)
    1: (4, 64, 32, 256, 4, "config1 tiny MM-DiT block (4 frames x 8x8 patches + 32 text, D256 H4)"),
    2: (16, 1350, 256, 1584, 24, "config2 Vchitect-2.0 2B block (16 frames x 30x45 patches + 256 text, D1584 H24)"),
    4: (160, 1350, 256, 1584, 24, "config4 long video 2B block (160 frames x 30x45 + 256 text)"),
    5: (64, 256, 256, 3072, 24, "config5 temporal-dominant block (64 frames x 16x16 + 256 text, D3072 H24)"),
}
METRIC = "video tokens/sec per denoise step (2B block, bf16)"


def algorithmic_flops(F, Lv, Lt, D, H):
    """per-kernel algorithmic FLOPs (no padding, text keys deduplicated)."""
    Nv = F * Lv
    return {
        "qkv_gemm": 2.0 * D * (9 * D * Nv + 2 * D * Lt),
        "attn_spatial": 4.0 * F * Lv * Lv * D,
        "attn_temporal": 4.0 * Lv * F * F * D,
        "attn_fullseq": 4.0 * Nv * (Nv + Lt) * D,
        "oproj_gemm": 2.0 * Nv * 3 * D * D,
    }


def algorithmic_bytes(F, Lv, Lt, D, H):
    Nv = F * Lv
    return {"ln": (Nv + Lt) * D * (4 + 2)}


def tensor_peak(peaks, clocks):
    """The bf16 roofline denominator for a kernel timed inside this run: the
    burst peak when the SM clock stayed at its maximum through the timed
    region (MEASURED_PEAKS.json bf16_tflops), the sustained one when it did
    not (a power-capped multi-second run)."""
    sm, mx = (clocks or {}).get("sm_mhz"), (clocks or {}).get("sm_max_mhz")
    if sm and mx and sm >= 0.97 * mx:
        return peaks["tc"], f"{peaks['src']} bf16 burst (SM clock at its maximum during the timed region)"
    return peaks["tc_sus"], f"{peaks['src']} bf16 sustained (SM clock below its maximum during the timed region)"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm": d.get("hbm_gbs", 6650.0), "tc": d.get("bf16_tflops", 1590.0),
                "tc_sus": d.get("bf16_tflops_sustained", 1400.0), "src": "measured"}
    return {"hbm": 6650.0, "tc": 1590.0, "tc_sus": 1400.0, "src": "fallback"}


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled DURING the timed region.

    NVML polled from a thread every ~2 ms (a timed region of a few tens of ms
    still gets many samples); `nvidia-smi -lms` is the fallback when NVML is
    missing. The device is matched by PCI bus id, so CUDA_VISIBLE_DEVICES
    remapping cannot point the sampler at another GPU."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.sw_power_cap",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown"]
    NAMES = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]

    def __init__(self, index=0, period_s=0.002):
        self.index = index
        self.period = period_s
        self.proc = None
        self.nvml = None
        self.samples = []  # (sm_mhz, max_mhz, {reasons})
        self.lines = []
        self.stop = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _sample_nvml(self):
        nv, h = self.nvml
        bits = {"sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                "hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown}
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.samples.append((float(sm), float(mx), {k for k, b in bits.items() if r & b}))

    def _poll_nvml(self):
        while True:
            self._sample_nvml()
            if self.stop.wait(self.period):
                break

    def __enter__(self):
        try:
            self.nvml = self._nvml_handle()
            self.thread = threading.Thread(target=self._poll_nvml, daemon=True)
            self.thread.start()
            # the poller is running before the timed region starts: wait for its
            # first sample, then drop it (it predates the region)
            t0 = time.time()
            while not self.samples and time.time() - t0 < 2.0:
                time.sleep(0.0005)
            self.samples.clear()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.thread.join(timeout=5)
            if not self.samples:  # a region shorter than one poll: sample at its end
                self._sample_nvml()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        samples = list(self.samples)
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                samples.append((float(parts[0]), float(parts[1]),
                                {n for n, v in zip(self.NAMES, parts[2:]) if v.lower().startswith("active")}))
            except ValueError:
                continue
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = set().union(*(r for _, _, r in samples))
        return {"sm_mhz": float(np.median([s for s, _, _ in samples])),
                "sm_max_mhz": max(m for _, m, _ in samples), "reasons": sorted(reasons),
                "samples": len(samples), "source": "nvml" if self.samples else "nvidia-smi"}


# ---------------------------------------------------------------------------
# CPU baseline: the pinned oracle port, exact frame slices of the block
# ---------------------------------------------------------------------------

def cpu_slices(cfg_id, seed=2025):
    """The reference block forward of the config's clip (oracle port, fp64),
    ready to run frame slice by frame slice (oracle/frame_slices.py: F
    consecutive slices are exactly one block forward's arithmetic)."""
    from oracle import spsim_oracle as O
    from oracle.frame_slices import FrameSlices
    F, Lv, Lt, D, H, _ = CONFIGS[cfg_id]
    blk = O.BlockParams.init(O.SeededRng(seed).split(1000), D)
    data = O.SeededRng(seed).split(1 << 20)
    x = data.split(1).normal((F, Lv, D))
    prompt = data.split(2).normal((Lt, D))
    return FrameSlices(blk, x, prompt, H)


def time_slices(fs, n, start=0):
    """Run n consecutive frame slices; returns the per-slice seconds."""
    out = []
    for i in range(n):
        t0 = time.perf_counter()
        fs.step((start + i) % fs.F)
        out.append(time.perf_counter() - t0)
    return out


def slice_sample_text(cfg_id, n):
    F, Lv, Lt, D, H, name = CONFIGS[cfg_id]
    return (f"oracle port of the reference block forward (fp64 numpy, pinned to the reference's golden outputs), "
            f"{name}: {n} exact frame slices (one slice = 1/{F} of the block's arithmetic: frame f's spatial "
            f"sequence, its rows' temporal queries against all {F} frames, its {Lt}+{Lv} full-sequence queries "
            f"against all {F * (Lt + Lv)} keys, each slice re-projecting its own frame's K/V), "
            f"{Lv} visual tokens per slice; tokens/s = slices x {Lv} / their total time")


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.config not in CONFIGS:
        print(json.dumps({"impl": "reference", "unavailable":
                          "the reference arm times block configs (1, 2, 4, 5); config 3 is a 40-block model step"}))
        return
    F, Lv, Lt, D, H, name = CONFIGS[args.config]
    fs = cpu_slices(args.config)
    time_slices(fs, args.warmup)
    ts = time_slices(fs, args.steps, start=args.warmup)
    total = float(sum(ts))
    value = args.steps * Lv / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SeededRng)",
        "config": {"workload": name, "frames": F, "visual_len": Lv, "text_len": Lt, "dim": D,
                   "heads": H, "tokens_per_step": Lv,
                   "step": f"one exact 1/{F} frame slice of the block forward ({Lv} visual tokens)"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cpu_cores(), "kind": "port",
                         "sample": slice_sample_text(args.config, args.steps)},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def make_inputs(torch, cfg_id, D, H, dtype, seed=2025, return_block=False):
    import paper_2501_08453_b200 as vc
    from paper_2501_08453_b200.model import DeviceBlock
    F, Lv, Lt = CONFIGS[cfg_id][:3]
    g = torch.Generator(device="cuda").manual_seed(seed)
    blk = vc.BlockParams.init(vc.SeededRng(seed).split(1000), D)  # random-init 2B-shape weights
    db = DeviceBlock(torch, blk, H, dtype)
    x = torch.randn((F, Lv, D), device="cuda", generator=g)
    prompt = torch.randn((Lt, D), device="cuda", generator=g)
    if return_block:
        return db, x, prompt, blk
    return db, x, prompt


def stage_profile(torch, lib, fwd, reps):
    lib.vc_profile_reset()
    lib.vc_profile_enable(1)
    for _ in range(reps):
        fwd()
    torch.cuda.synchronize()
    lib.vc_profile_enable(0)
    ms = (C.c_double * 32)()
    calls = (C.c_int32 * 32)()
    names = C.create_string_buffer(2048)
    n = lib.vc_profile_read(ms, calls, 32, names, 2048)
    out = {}
    for i, nm in enumerate(names.value.decode().split("\n")[:n]):
        out[nm] = ms[i] / max(calls[i], 1)
    return out


def run_gpu_arm(args):
    import torch
    import paper_2501_08453_b200 as vc  # noqa: F401
    from paper_2501_08453_b200 import _lib
    from paper_2501_08453_b200.model import block_forward_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if args.config == 3:
        return run_model_step(args, torch, world, rank, local)
    if world > 1 or args.sp:
        return run_gpu_sp(args, torch, world, rank, local)

    lib = _lib.load()
    F, Lv, Lt, D, H, name = CONFIGS[args.config]
    Nv = F * Lv
    db, x, prompt = make_inputs(torch, args.config, D, H, args.dtype)
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def fwd():
        block_forward_device(torch, db, x, prompt, out, False)

    for _ in range(max(args.warmup, 3)):
        fwd()
    torch.cuda.synchronize()
    # ---- timed region (device, CUDA events on the launching stream) ----
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            fwd()
        e1.record(stream)
        torch.cuda.synchronize()
    ms_per_step = e0.elapsed_time(e1) / args.steps
    value = Nv / (ms_per_step / 1e3)

    # ---- end to end through the public serving API with pinned HOST buffers ----
    # block_forward_host_stream -> vc_block_forward_host_batched: every step
    # copies its input H2D and its result D2H; the copies of neighbouring
    # steps overlap the compute of this one (double-buffered staging).
    from paper_2501_08453_b200.model import block_forward_host_stream
    shp = _lib.shape(F, Lv, Lt, D, H, args.dtype)
    xh = [x.cpu().pin_memory() for _ in range(2)]
    ph = prompt.cpu().pin_memory()
    inputs = [xh[i % 2] for i in range(args.steps)]
    outs = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
    out_list = [outs[i % 2] for i in range(args.steps)]
    # the serving handle: weights already packed on the device (DeviceBlock)
    block_forward_host_stream(db, inputs[:3], ph, H, out_list[:3])  # warm-up
    torch.cuda.synchronize()
    e0.record(stream)
    block_forward_host_stream(db, inputs, ph, H, out_list)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    oh = out_list[-1]
    assert torch.isfinite(oh).all().item()
    single_host_ms = None
    hws = lib.vc_block_host_workspace_bytes(C.byref(shp))
    if hws:
        ws1 = torch.empty(hws, dtype=torch.uint8, device="cuda")
        e0.record(stream)
        for _ in range(3):
            _lib.check(lib.vc_block_forward_host(C.byref(shp), _lib.ptr(db.packed), C.c_void_p(xh[0].data_ptr()),
                                                 C.c_void_p(ph.data_ptr()), C.c_void_p(outs[0].data_ptr()),
                                                 _lib.ptr(ws1), hws, _lib.stream_ptr(torch)), "forward_host")
        e1.record(stream)
        torch.cuda.synchronize()
        single_host_ms = e0.elapsed_time(e1) / 3
        del ws1

    # ---- per-stage device time (separate, untimed pass) ----
    stages = stage_profile(torch, lib, fwd, max(2, min(args.steps, 5)))
    flops = algorithmic_flops(F, Lv, Lt, D, H)
    peaks = load_peaks()
    dom = max((k for k in stages if k in flops), key=lambda k: stages[k])
    achieved = flops[dom] / (stages[dom] / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"cfg{args.config}_{args.dtype}", {}).get(dom)
    block_tflops = sum(flops.values()) / (ms_per_step / 1e3) / 1e12

    cpu = None
    if not args.no_cpu_baseline:
        fs = cpu_slices(args.config)
        ts = time_slices(fs, 2)
        cpu = {"value": 2 * Lv / sum(ts), "unit": "tokens/s", "cores": cpu_cores(), "kind": "port",
               "sample": slice_sample_text(args.config, 2)}

    launches = lib.vc_block_forward_launches(C.byref(shp)) * args.steps
    clocks = clk.summary()
    peak, peak_kind = tensor_peak(peaks, clocks)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (torch.randn inputs, SeededRng random-init 2B-shape weights)",
        "config": {"workload": name, "frames": F, "visual_len": Lv, "text_len": Lt, "dim": D,
                   "heads": H, "tokens_per_step": Nv, "parallelism": "single GPU",
                   "l2": "inputs larger than L2 (x fp32 %.0f MB + weights %.0f MB > 126 MB)"
                   % (Nv * D * 4 / 1e6, db.packed.numel() / 1e6)},
        "roofline": {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "share_of_step": stages[dom] / sum(stages.values())},
        "block": {"tflops_algorithmic": block_tflops, "frac_of_bf16_peak": block_tflops / peaks["tc"],
                  "frac_of_bf16_sustained": block_tflops / peaks["tc_sus"],
                  "peak_note": "frac_of_bf16_peak is against the burst peak (MEASURED_PEAKS.json bf16_tflops)",
                  "stage_ms": stages, "stage_sum_ms": sum(stages.values())},
        "cpu_baseline": cpu,
        "e2e": {"value": Nv / (e2e_ms / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": Nv * D * 4, "d2h_bytes_per_step": Nv * D * 4,
                "api": "paper_2501_08453_b200.model.block_forward_host_stream (vc_block_forward_host_batched) on "
                       "the device-resident weight handle, %d steps in one call, pinned host in/out, copies "
                       "overlapped across steps (pipeline fill + drain inside the timed region)" % args.steps,
                "single_call_tokens_per_s": Nv / (single_host_ms / 1e3) if single_host_ms else None},
        "clocks": clocks,
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)


def run_model_step(args, torch, world, rank, local):
    """Config 3: one full 2B-model denoise step (ToyDenoiser.forward: embed +
    40 blocks + unembed, model.py:327-333) on a 480p 40-frame latent clip;
    sequence-parallel over the ranks when world > 1 (sp.sp_model_forward)."""
    import paper_2501_08453_b200 as vc
    from paper_2501_08453_b200 import sp
    F, h, w, Lt, D, H, depth = 40, 60, 90, 256, 1584, 24, args.depth
    name = f"config3 2B ToyDenoiser step ({depth} blocks, 40 frames x 60x90 latents -> 30x45 patches, 256 text)"
    Lv = (h // 2) * (w // 2)
    Nv = F * Lv
    model = vc.ToyDenoiser.init(vc.SeededRng(2025), vc.PatchSpec(8, 2, 4), D, H, depth)
    g = torch.Generator(device="cuda").manual_seed(2025)
    lat = torch.randn((F, h, w, 4), device="cuda", generator=g)
    prompt = torch.randn((Lt, D), device="cuda", generator=g)
    stream = torch.cuda.current_stream()
    if world > 1 or args.sp:
        import torch.distributed as dist
        for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29541"), ("RANK", "0"), ("WORLD_SIZE", "1")):
            os.environ.setdefault(k, v)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        cache, ex = {}, sp.TorchExchange()

        def step():
            return sp.sp_model_forward(torch, model, lat, 37, prompt, cache, ex, rank, world)
        par = f"sequence parallel sp{world} (own-row embed, head-parallel a2a per block, final all-gather)"
    else:
        def step():
            return model.forward(lat, 37, prompt, dtype="bf16")
        par = "single GPU"
    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1 or args.sp:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            eps = step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    if world > 1 or args.sp:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_per_step = float(ms.item())
    assert torch.isfinite(eps).all().item()
    flops = depth * sum(algorithmic_flops(F, Lv, Lt, D, H).values())
    peaks = load_peaks()
    clocks = clk.summary()
    peak, peak_kind = tensor_peak(peaks, clocks)
    if rank == 0:
        line = {
            "metric": METRIC, "value": Nv / (ms_per_step / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 1), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic latents/prompt, SeededRng random-init 2B weights",
            "config": {"workload": name, "frames": F, "visual_len": Lv, "text_len": Lt, "dim": D, "heads": H,
                       "depth": depth, "tokens_per_step": Nv, "parallelism": par},
            "roofline": {"bound": "tensor", "kernel": "whole model step (per GPU)",
                         "achieved": flops / world / (ms_per_step / 1e3) / 1e12, "peak": peak,
                         "unit": "TFLOP/s", "frac": flops / world / (ms_per_step / 1e3) / 1e12 / peak,
                         "traffic": None, "peak_kind": peak_kind},
            "cpu_baseline": None, "e2e": None, "clocks": clocks, "gpu_launches": None,
        }
        print(json.dumps(line), flush=True)
    if world > 1 or args.sp:
        dist.barrier()
        dist.destroy_process_group()


def run_gpu_sp(args, torch, world, rank, local):
    from paper_2501_08453_b200 import sp
    return sp.bench_sp(args, torch, world, rank, local, CONFIGS, METRIC, algorithmic_flops,
                       load_peaks, tensor_peak, ClockSampler, cpu_slices, time_slices, slice_sample_text,
                       cpu_cores, stage_profile)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS) + [3])
    ap.add_argument("--depth", type=int, default=40, help="blocks in the config-3 model step")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--sample-frames", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sp", action="store_true",
                    help="run the sequence-parallel (NCCL) path even at world size 1")
    ap.add_argument("--sp-mode", default="head_parallel", choices=["head_parallel", "gather"],
                    help="SP attention: head-parallel all-to-alls (default) or K/V all-gather "
                         "(chosen automatically when the GPU count does not divide the heads)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return run_gpu_arm(args)


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-launch this command as N
    ranks, one per GPU (torch.distributed.run, 127.0.0.1 rendezvous); rank 0
    prints the line."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} GPU(s) visible")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    raise SystemExit(subprocess.call(cmd))


if __name__ == "__main__":
    main()
