#!/usr/bin/env python
"""SpecFormer decode-step benchmark (one JSON line on rank 0).

A "step" = one draft_step + verify_step + accept_commit over the GPU's batch (all §8(a) rows),
replayed from a CUDA graph through the C ABI. Workload: BASELINE.json configs[2] (7B-shaped,
k = 4, prompt 512) at batch 64 per GPU (weak scaling across ranks); synthetic seeded weights and
uniform-random prompts; inputs (14 GB of weights + KV) are far larger than the 126 MB L2, so no
explicit flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--config 7b] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, max-over-ranks timing)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

A_PAPER = {"small": 1.84, "7b": 1.75, "13b": 1.71, "70b": 1.71, "tiny": 1.84}  # SURVEY §8d (T3, k=4)
METRIC = "generated tokens/s per box (7B-shaped SpecFormer SD step, measured acceptance)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons DURING the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, dev_index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()
        self.active = True  # start() / stop() restrict the samples to the timed windows

    def start(self):
        self.active = True

    def stop(self):
        self.active = False

    def _run(self):
        while not self._stop.is_set():
            if not self.active:
                time.sleep(0.002)
                continue
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        self.active = False
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- oracle leg
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(cfg, n_steps=2, prompt_len=None, threads=None):
    """Time the fp64 oracle (as it stands, never tuned) on a bounded sample of the workload: ONE
    sequence at the config's full width and prompt length (512 for the 7B shape) with the base
    truncated to L = 1 and L = 2 layers (the SpecFormer head unchanged). For each depth,
    oracle.sd_decode runs the prefill and n_steps decode steps; the mean wall time of those steps
    (oracle step_times hook) is the measured per-step time at that depth. Full depth is an
    EXTRAPOLATION, linear in L: t(L) = t(1) + (L - 1) (t(2) - t(1)). The
    oracle computes sequences one at a time, so box tokens/s = tokens per step / t(L_full).
    `threads`: BLAS threads (None = every core of the affinity mask; 1 = the single-thread figure)."""
    import oracle as O
    from synth import make_prompts, make_weights

    P = cfg.prompt_len if prompt_len is None else prompt_len
    c2 = cfg.replace(n_layers=2)
    w = make_weights(c2, seed=0, device="cpu")
    prompt = make_prompts(1, P, cfg.vocab)[0].tolist()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    nthr = cores if threads is None else threads
    try:
        from threadpoolctl import threadpool_limits
        limit = threadpool_limits(limits=nthr)
    except Exception:  # pragma: no cover - threadpoolctl is in the image
        limit = None
    times, toks, steps_run, secs_run = {}, {}, 0, 0.0
    try:
        for L in (1, 2):
            W = O.Weights(cfg.replace(n_layers=L), w)
            O.sd_decode(W, prompt[:8], 2)  # warm the fp64 weight cache (upcast) outside the timing
            st_times = []
            _, st = O.sd_decode(W, prompt, 1 + n_steps, step_times=st_times)  # prefill, then n_steps steps
            times[L] = sum(st_times) / len(st_times)
            toks[L] = sum(s_["m"] + 1 for s_ in st) / max(1, len(st))
            steps_run += len(st_times)
            secs_run += sum(st_times)
    finally:
        if limit is not None and hasattr(limit, "unregister"):
            limit.unregister()
    t_full = times[1] + (cfg.n_layers - 1) * max(0.0, times[2] - times[1])
    a = toks[2]
    return {"value": a / t_full, "unit": "tokens/s", "cores": nthr, "kind": "oracle", "cpu_model": cpu_model(),
            "extrapolated": True,
            "sample": f"1 sequence, width {cfg.d_model}, prompt {P}, base depth 1 and 2 of {cfg.n_layers} layers; "
                      f"measured per-step time t_step(L=1)={times[1]:.3f}s t_step(L=2)={times[2]:.3f}s "
                      f"(mean of {n_steps} decode steps after the untimed prefill), full depth EXTRAPOLATED "
                      f"linearly in L: t_step(L={cfg.n_layers})={t_full:.2f}s per sequence; sequences one at a "
                      f"time (numpy fp64, BLAS threads = {nthr}, {cpu_model()})",
            "seconds_per_step_per_sequence": t_full, "measured_steps": steps_run,
            "measured_ms_per_step": 1e3 * secs_run / max(1, steps_run),
            "measured_s_per_step_depth": {"1": times[1], "2": times[2]}}


def run_reference(args, cfg):
    """--impl reference: the fp64 oracle as it stands on the host cores, rank 0 only.
    ms_per_step is the time of the oracle steps that actually ran (depth-1 and depth-2 samples of one
    sequence); value is the labelled full-depth extrapolation in tokens/s."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t0 = time.perf_counter()
    cb = oracle_sample(cfg, n_steps=max(2, min(args.steps, 3)))
    cb1 = oracle_sample(cfg, n_steps=2, threads=1)  # the single-thread figure
    wall = time.perf_counter() - t0
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": cb["measured_steps"], "warmup": args.warmup,
            "ms_per_step": cb["measured_ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded N(0,0.02) weights, uniform-random prompts)",
            "config": {"workload": f"{cfg.name}-shaped SpecFormer decode step, batch {args.batch}/GPU, k {cfg.draft_len}",
                       "model": cfg.name, "batch_per_gpu": args.batch, "draft_len": cfg.draft_len,
                       "prompt_len": cfg.prompt_len, "l2": "inputs larger than L2"},
            "note": "steps / ms_per_step: the oracle steps actually run (one sequence, base depth 1 and 2); value: "
                    "full-depth tokens/s extrapolated linearly in depth (cpu_baseline.sample)",
            "cpu_baseline": cb,
            "cpu_baseline_1thread": cb1,
            "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU leg
def _log(msg):
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def run_ours(args, cfg):
    import ctypes as C

    import torch
    import torch.distributed as dist

    import numpy as np

    from paper_2511_20340_b200 import Engine, EngineConfig, dp, roofline, timeline
    from paper_2511_20340_b200 import tp as tpmod
    from paper_2511_20340_b200.engine import nccl_unique_id
    from synth.weights import weight_shapes
    from paper_2511_20340_b200 import _native as N
    from synth import make_prompts, make_weights

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B, k, P = args.batch, cfg.draft_len, cfg.prompt_len
    K, W = args.steps, args.warmup
    Kp = args.profile_steps
    Ke = args.e2e_steps if args.e2e_steps > 0 else cfg.gen_len - 1  # default: one full generation
    Kf = max(0, args.forced_steps) if k > 0 else 0
    n_cont = (W + Kf + 2) * (k + 1) + k + 2  # greedy-continuation tokens the forced window can consume
    # capacity: every phase restarts from a prefill; a decode_steps call of n steps needs n (k + 1)
    # positions of headroom over the actual length (a ~= 1 with random weights, so lengths grow ~1 per step)
    GEN_CHUNK = 16
    grow = max(W + K * (k + 1), W + K + (args.timeline_steps + Kp) * (k + 1), Ke + k + 1)
    if Kf:
        grow = max(grow, n_cont + GEN_CHUNK * (k + 1), (W + Kf) * (k + 1))
    max_seq = (P + grow + 32 + 15) // 16 * 16

    # --tp (default for the 70B shape): the ranks split one model (tensor parallelism, strong
    # scaling of one global batch B); otherwise each rank serves its own batch B (weak scaling)
    tp = world if (world > 1 and (args.tp or cfg.name == "70b")) else 1
    if cfg.name == "70b" and tp == 1:
        raise SystemExit("the 70B shape needs tensor parallelism: torchrun --nproc-per-node >= 2 (SURVEY 8e; "
                         "~141 GB of bf16 weights + KV do not fit one GPU)")
    if tp > 1:
        weights = tpmod.LazyWeights(lambda n: make_weights(cfg, seed=0, device="cuda", names={n})[n],
                                    [n for n, _ in weight_shapes(cfg)])
    else:
        weights = make_weights(cfg, seed=0, device="cuda")
    # the step consumes only the argmax of the logits: the bf16 LM heads fuse it and do not store them
    no_logits = cfg.dtype == "bf16" and not args.keep_logits
    ec = EngineConfig.from_model(cfg, max_batch=B, max_seq=max_seq,
                                 flags=N.SF_FLAG_CUDA_GRAPH | (N.SF_FLAG_NO_LOGITS if no_logits else 0),
                                 tp_size=tp, tp_rank=rank if tp > 1 else 0)
    eng = Engine(ec, weights)
    del weights
    torch.cuda.empty_cache()
    if tp > 1:
        eng.attach_nccl(tpmod.share_unique_id(nccl_unique_id, rank), tp, rank)
        if args.tp_fused:  # NEXT-3: row-parallel all-reduce fused into the norm consumer over peer memory
            eng.attach_xch(tpmod.share_xch_handles(eng.xch_handle(), rank, tp))
        prompts = make_prompts(B, P, cfg.vocab)  # every rank: the same global batch
    else:
        prompts = dp.shard_rows(make_prompts(B * world, P, cfg.vocab), rank, world)  # weak scaling

    n_win = max(1, args.windows)

    def timed_windows(Bs, prompts_s, clk=None):
        """n_win windows, each: prefill (untimed) + W warm-up steps + K timed steps of the captured step
        graph between CUDA events on the engine stream (barrier + sync on both sides); returns the window
        with the median time and every window's time."""
        wins = []
        acc = torch.zeros(max(K, W), Bs, dtype=torch.int32, device="cuda")
        for wi in range(n_win):
            _log(f"  window {wi}: prefill B={Bs}")
            eng.prefill(prompts_s.cuda())
            eng.sync()
            _log(f"  window {wi}: warm-up")
            eng.decode_steps(W, None, acc)  # warm-up; (re)captures the step graph the window replays
            eng.sync()
            b0 = eng.capture(3, (Bs,), torch.int32).cpu()
            p0 = eng.capture(5, (Bs,), torch.int32).cpu()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            if clk is not None:
                clk.start()
            torch.cuda.cudart().cudaProfilerStart()  # ncu --profile-from-start off: the timed windows only
            e0.record(eng.stream)
            eng.decode_steps(K, None, acc)
            e1.record(eng.stream)
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
            if clk is not None:
                clk.stop()
            if world > 1:
                dist.barrier()
            eng.sync()
            wms = e0.elapsed_time(e1)
            a1 = eng.capture(3, (Bs,), torch.int32).cpu()
            wins.append({"ms": wms, "before": b0, "prev_before": p0, "after": a1, "acc": acc.cpu().clone(),
                         "launches": eng.kernel_launches()})
        order = sorted(range(n_win), key=lambda i: wins[i]["ms"])
        med = dict(wins[order[n_win // 2]])
        med["all_ms"] = [w_["ms"] for w_ in wins]
        return med

    def window_roofline(win, Bs):
        lens_t, prev_t, accs_t = win["before"].tolist(), win["prev_before"].tolist(), win["acc"].tolist()
        sb_ = 0.0
        for s_ in range(K):
            sb_ += roofline.step_bytes(cfg, Bs, k, lens_t, prev_t, logits=not no_logits)
            prev_t = list(lens_t)
            lens_t = [n + m + 1 for n, m in zip(lens_t, accs_t[s_])]
        return sb_ / tp

    _log(f"timed windows B={B}")
    with ClockSampler(local) as clk:
        main = timed_windows(B, prompts, clk)
    ms = main["ms"]
    launches = main["launches"]
    before, prev_before, after = main["before"], main["prev_before"], main["after"]
    acc_log = main["acc"].cuda()
    tokens = int((after - before).sum())
    ms_max, tokens_total = dp.reduce_timing(ms, float(tokens), device="cuda")
    tokens_total /= tp  # tensor parallelism: every rank emits the same tokens
    value = tokens_total / (ms_max / 1e3)
    steps_per_s = K / (ms_max / 1e3)
    a_meas = tokens / (K * B)

    # ---------------- whole-step roofline over the timed (graph) region, lengths from the accept log
    sb = window_roofline(main, B)  # (tensor parallelism: each GPU streams 1/tp of the weights / KV heads)
    step_gbs = sb / (ms / 1e3) / 1e9

    def replay_lengths(lens0, prev0, accs, Bs):
        """algorithmic KV bytes / step bytes / step flops of the steps whose accept rows are accs"""
        lens, prevs, kv, by, fl = list(lens0), list(prev0), 0.0, 0.0, 0.0
        for a in accs:
            kv += roofline.attention_kv_bytes(cfg, lens, prevs, k)
            by += roofline.step_bytes(cfg, Bs, k, lens, prevs, logits=not no_logits)
            fl += roofline.step_flops(cfg, Bs, k, lens)
            prevs = list(lens)
            lens = [n + m + 1 for n, m in zip(lens, a)]
        return kv, by, fl

    hbm, tf_burst, tf_sust, peak_src0 = peaks()
    d_, F_, V_ = cfg.d_model, cfg.d_ff, cfg.vocab
    qkv_ = (cfg.n_heads + 2 * cfg.n_kv_heads) * cfg.head_dim
    ao_ = cfg.n_heads * cfg.head_dim

    def gemm_flops(Bs):
        """GEMM FLOPs of one step (2 T N K summed over the step's contractions)"""
        Tv, Td = Bs * (k + 1), Bs * k
        per_layer = qkv_ * d_ + d_ * ao_ + 2 * F_ * d_ + d_ * F_
        return 2.0 * (Tv * (cfg.n_layers * per_layer + V_ * d_) + Tv * (4 * d_ * d_ + qkv_ * d_ + d_ * ao_)
                      + Bs * k * d_ * d_ + Td * (qkv_ * d_ + d_ * ao_ + 3 * F_ * d_ + V_ * d_)) / tp

    def event_profile(Bs):
        """Kp steps of the step graph re-captured with a CUDA event-record node around every launch (on
        the engine stream: the launches' own stream), replayed one step at a time; per kernel class:
        time, launches, algorithmic bytes (GEMM: host-known weights + activations + outputs; attention:
        KV bytes from the accept log). The record nodes serialise the launches (no PDL overlap), so these
        per-launch times are conservative. Also picks the dominant class and its roofline."""
        lens0 = eng.capture(3, (Bs,), torch.int32).cpu().tolist()
        prev0 = eng.capture(5, (Bs,), torch.int32).cpu().tolist()  # context layer runs at n_prev
        acc_p = torch.zeros(Kp, Bs, dtype=torch.int32, device="cuda")
        eng.profile(True)
        ep0, ep1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ep0.record(eng.stream)
        eng.decode_steps(Kp, None, acc_p)
        ep1.record(eng.stream)
        eng.sync()
        tot = ep0.elapsed_time(ep1)
        cls = {c: eng.profile_read(c) for c in range(4)}
        eng.profile(False)
        attn_bytes, _, step_flops_tot = replay_lengths(lens0, prev0, acc_p.cpu().tolist(), Bs)
        attn_bytes /= tp
        gemm_ms, gemm_n, gemm_bytes = cls[0]
        attn_ms, attn_n, _ = cls[1]
        gf = gemm_flops(Bs)
        classes = {name: {"ms_total": cls[c][0], "launches": cls[c][1], "share_of_profiled_step":
                          cls[c][0] / max(1e-9, tot)}
                   for c, name in enumerate(["gemm", "attention", "norm", "argmax"])}
        g_gbs = gemm_bytes / max(1e-12, gemm_ms / 1e3) / 1e9
        g_tfs = gf * Kp / max(1e-12, gemm_ms / 1e3) / 1e12
        a_gbs = attn_bytes / max(1e-12, attn_ms / 1e3) / 1e9
        g_bound_tc = gf / (tf_sust * 1e12) > (gemm_bytes / Kp) / (hbm * 1e9)
        classes["gemm"].update(achieved_gbs=g_gbs, achieved_tflops=g_tfs, bound="tensor" if g_bound_tc else "hbm",
                               frac=(g_tfs / tf_sust) if g_bound_tc else (g_gbs / hbm),
                               bytes_per_step=gemm_bytes / Kp, flops_per_step=gf)
        classes["attention"].update(achieved_gbs=a_gbs, frac=a_gbs / hbm, bytes_per_step=attn_bytes / Kp)
        dominant = "gemm" if gemm_ms >= attn_ms else "attention"
        n_dom = (gemm_n if dominant == "gemm" else attn_n) / max(1, Kp)
        dom_ms = (gemm_ms if dominant == "gemm" else attn_ms) / max(1, Kp) / max(1e-9, n_dom)
        if dominant == "gemm" and g_bound_tc:
            bound, unit, peak_v, units = "tensor", "TFLOP/s", tf_sust, gf / max(1e-9, n_dom)
            psrc = peak_src0 + " (bf16_tflops_sustained: kernel timed inside the step)"
            achieved = units / (dom_ms / 1e3) / 1e12
        else:
            bound, unit, peak_v, psrc = "hbm", "GB/s", hbm, peak_src0 + " (hbm_gbs)"
            units = (gemm_bytes if dominant == "gemm" else attn_bytes) / max(1, Kp) / max(1e-9, n_dom)
            achieved = units / (dom_ms / 1e3) / 1e9
        return {"classes": classes, "profiled_steps": Kp, "profiled_ms_total": tot, "dominant": dominant,
                "bound": bound, "unit": unit, "peak": peak_v, "peak_source": psrc, "achieved": achieved,
                "frac": achieved / peak_v, "units_per_launch": units, "ms_per_launch": dom_ms,
                "launches_per_step": n_dom, "step_flops": step_flops_tot / max(1, Kp)}

    def e2e_run(Bs, prompts_s, n_steps):
        """One generation through the public C ABI: prompt H2D from pinned host memory, prefill, then per
        step one specformer_decode_steps(1) call (the captured step graph) followed by the D2H read of that
        step's accept lengths and emitted tokens into pinned host buffers; all inside the events."""
        lib = eng.lib
        host_prompts = prompts_s.clone().pin_memory()
        g_host = torch.empty(Bs, dtype=torch.int32).pin_memory()
        m_host = torch.empty(n_steps, Bs, dtype=torch.int32).pin_memory()
        em_host = torch.empty(n_steps, Bs, k + 1, dtype=torch.int32).pin_memory()
        em_dev = torch.empty(1, Bs, k + 1, dtype=torch.int32, device="cuda")
        m_dev = torch.empty(1, Bs, dtype=torch.int32, device="cuda")
        p = lambda t: C.c_void_p(t.data_ptr())
        st = lib.specformer_prefill(eng.h, p(host_prompts), Bs, P, p(g_host))  # warm-up: captures the step graph
        for _ in range(2):
            st |= lib.specformer_decode_steps(eng.h, 1, p(em_dev), p(m_dev))
        eng.sync()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(eng.stream)
        st |= lib.specformer_prefill(eng.h, p(host_prompts), Bs, P, p(g_host))
        with torch.cuda.stream(eng.stream):  # the D2H copies run on the engine stream, after each step
            for s_ in range(n_steps):
                st |= lib.specformer_decode_steps(eng.h, 1, p(em_dev), p(m_dev))
                em_host[s_].copy_(em_dev[0], non_blocking=True)
                m_host[s_].copy_(m_dev[0], non_blocking=True)
        x1.record(eng.stream)
        eng.sync()
        if st != 0:
            raise RuntimeError("e2e C-ABI call failed")
        e_ms = x0.elapsed_time(x1)
        e_tok = Bs + int((em_host >= 0).sum())
        e_ms_max, e_tok = dp.reduce_timing(e_ms, float(e_tok), device="cuda")
        e_tok /= tp
        return {"value": e_tok / (e_ms_max / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": Bs * P * 4 / n_steps, "d2h_bytes_per_step": Bs * (k + 2) * 4,
                "steps": n_steps, "includes_prefill": True,
                "note": "one generation through the public C ABI with pinned host buffers: prompt H2D + prefill + "
                        "per-step specformer_decode_steps(1) calls (draft + verify + accept, replayed from the "
                        "step's CUDA graph), each step's accept lengths / emitted tokens copied to the host; "
                        "prompt bytes amortised over the steps"}

    # ---------------- kernel timeline (secondary): Kt replays of the timed step graph with the per-CTA
    # %globaltimer probes on; the step's critical path attributed to kernel classes (credits PDL overlap)
    Kt = args.timeline_steps
    tl = None
    if Kt > 0 and N.lib().sf_debug_ktrace_enable(1) == 0:
        _log("timeline")
        lt0 = eng.capture(3, (B,), torch.int32).cpu().tolist()
        pt0 = eng.capture(5, (B,), torch.int32).cpu().tolist()
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0e.record(eng.stream)
        eng.decode_steps(Kt, None, acc_log)  # the same graph the timed window replayed
        t1e.record(eng.stream)
        eng.sync()
        buf = np.zeros(1 << 21, dtype=timeline.REC)
        n_rec = N.lib().sf_debug_ktrace(C.c_void_p(buf.ctypes.data), buf.size)
        N.lib().sf_debug_ktrace_enable(0)
        cp = timeline.critical_path(buf[:n_rec], key=timeline.kclass)
        kv_t, _, _ = replay_lengths(lt0, pt0, acc_log[:Kt].cpu().tolist(), B)
        tl = {"steps": Kt, "cta_records": int(n_rec), "events_ms_per_step": t0e.elapsed_time(t1e) / Kt,
              "span_ms_per_step": cp["span_us"] / 1e3 / Kt, "idle_gap_ms_per_step": cp["gap_us"] / 1e3 / Kt,
              "classes": {c: {"exposed_ms_per_step": cp["exposed"][c] / 1e3 / Kt,
                              "launches_per_step": cp["count"][c] / Kt,
                              "share_of_step": cp["exposed"][c] / max(1e-9, cp["span_us"])}
                          for c in cp["exposed"]},
              "attention_kv_bytes": kv_t}
        g_tl = tl["classes"].get("gemm")
        if g_tl:
            g_ms = g_tl["exposed_ms_per_step"] / max(1e-9, g_tl["launches_per_step"])
            tl["gemm_tflops_exposed"] = gemm_flops(B) / max(1e-9, g_tl["launches_per_step"]) / (g_ms / 1e3) / 1e12

    _log("event profile")
    ev = event_profile(B)
    dominant = ev["dominant"]
    # DRAM bytes per launch of the dominant kernel class from the committed ncu launch list of this
    # command at this batch (profiles/ncu_traffic.json, written by tools/profile_summary.py)
    traffic = None
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(traffic_path):
        try:
            traffic = json.load(open(traffic_path)).get(f"{cfg.name}_b{B}", {}).get("traffic_bytes_per_launch", {}).get(dominant)
        except Exception:
            traffic = None
    _log("e2e")
    e2e = e2e_run(B, prompts, Ke)
    _log("prefill")

    # ---------------- prefill (untimed in the decode metric; NEXT-4): chunked base forward +
    # context layer over the B x P prompt rows, timed with CUDA events on the engine stream
    pf_ms = []
    for _ in range(2):
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        q0.record(eng.stream)
        eng.prefill(prompts.cuda())
        q1.record(eng.stream)
        eng.sync()
        pf_ms.append(q0.elapsed_time(q1))
    c_pf = max(k + 1, min(512, max(1, 512 // B)))
    n_chunks = -(-P // c_pf)
    pf_flops = roofline.prefill_flops(cfg, B, P, k) / tp
    pf_bytes = roofline.prefill_bytes(cfg, B, P, k, n_chunks) / tp
    pms = min(pf_ms)
    pf_tc = pf_flops / (pms / 1e3) / 1e12
    prefill = {"ms": pms, "tokens_per_s": B * P / (pms / 1e3), "chunks": n_chunks, "rows_per_chunk": B * c_pf,
               "flops": pf_flops, "bytes": pf_bytes, "achieved_tflops": pf_tc, "frac_tensor_sustained": pf_tc / tf_sust,
               "achieved_gbs": pf_bytes / (pms / 1e3) / 1e9,
               "t_roof_ms": 1e3 * max(pf_flops / (tf_sust * 1e12), pf_bytes / (hbm * 1e9)),
               "frac_roofline": 1e3 * max(pf_flops / (tf_sust * 1e12), pf_bytes / (hbm * 1e9)) / pms}

    # ---------------- batch sweep (BASELINE metric: verify-steps/s vs batch 1-64): the same engine
    # re-prefilled at each smaller batch; per batch the median of the timed windows, the step
    # roofline, event-timed GEMM / attention fractions and one end-to-end generation
    sweep = []
    for Bs in args.sweep_list:
        if Bs >= B or tp > 1:
            continue
        _log(f"sweep B={Bs}")
        pr_s = prompts[:Bs].contiguous()
        with ClockSampler(local) as clk_s:
            win = timed_windows(Bs, pr_s, clk_s)
        sb_s = window_roofline(win, Bs)
        w_ms, w_tok = dp.reduce_timing(win["ms"], float(int((win["after"] - win["before"]).sum())), device="cuda")
        _log("  event profile")
        ev_s = event_profile(Bs)
        _log("  e2e")
        sweep.append({"batch_per_gpu": Bs, "value": w_tok / (w_ms / 1e3), "unit": "tokens/s",
                      "ms_per_step": w_ms / K, "window_ms": win["all_ms"],
                      "verify_steps_per_s": K / (w_ms / 1e3), "mean_accepted_length": w_tok / (K * Bs * world),
                      "step_roofline": {"bound": "hbm", "achieved": sb_s / (win["ms"] / 1e3) / 1e9, "peak": hbm,
                                        "unit": "GB/s", "frac": sb_s / (win["ms"] / 1e3) / 1e9 / hbm,
                                        "bytes_per_step": sb_s / K, "t_roof_ms": (sb_s / K) / (hbm * 1e9) * 1e3},
                      "roofline": {k_: ev_s[k_] for k_ in ("bound", "achieved", "peak", "unit", "frac", "peak_source",
                                                           "ms_per_launch", "launches_per_step")} | {"kernel": ev_s["dominant"]},
                      "event_classes": ev_s["classes"],
                      "e2e": e2e_run(Bs, pr_s, min(Ke, args.sweep_e2e_steps)),
                      "clocks": clk_s.summary(),
                      "gpu_launches": win["launches"]})

    # ---------------- forced acceptance: drafts replaced -- after the draft step has run
    # and been paid for -- by the GPU's own greedy continuation, corrupted at slot j with
    # P(j) = alpha^(j-1) (1 - alpha) (none with alpha^k), alpha set so E[tokens/step] = a_paper
    forced = None
    if Kf:
        _log("forced acceptance")
        a_target = A_PAPER.get(cfg.name, 1.75)
        lo, hi = 0.0, 0.999
        for _ in range(60):
            mid = (lo + hi) / 2
            if (1 - mid ** (k + 1)) / (1 - mid) < a_target: lo = mid
            else: hi = mid
        alpha = (lo + hi) / 2
        # the continuation: lossless SD with measured acceptance emits the greedy sequence
        g0 = eng.prefill(prompts.cuda())
        n_gen = n_cont
        em_log = torch.full((n_gen, B, k + 1), -1, dtype=torch.int32, device="cuda")
        for s0 in range(0, n_gen, GEN_CHUNK):  # chunked: each call needs only GEN_CHUNK (k+1) of headroom
            eng.decode_steps(min(GEN_CHUNK, n_gen - s0), em_log[s0:], None)
        eng.sync()
        em = em_log.cpu()
        cont = torch.zeros(B, n_cont, dtype=torch.int32)
        g0c = g0.cpu()
        for b in range(B):
            toks = [int(g0c[b])] + [int(t) for t in em[:, b, :].reshape(-1) if int(t) >= 0]
            toks = (toks + [toks[-1]] * n_cont)[:n_cont]
            cont[b] = torch.tensor(toks, dtype=torch.int32)
        gen = torch.Generator().manual_seed(2)  # per (step, global sequence): identical at any GPU count
        n_cs = W + Kf + 2
        nb = B if tp > 1 else B * world  # (tensor parallelism: one batch, the same on every rank)
        r0 = 0 if tp > 1 else rank * B
        u = torch.rand(n_cs, nb, generator=gen)[:, r0:r0 + B]
        cdf = torch.tensor([sum(alpha ** (i - 1) * (1 - alpha) for i in range(1, j + 1)) for j in range(1, k + 1)])
        corrupt = (torch.searchsorted(cdf, u.contiguous()) + 1).to(torch.int32)  # k + 1 = no corruption
        eng.prefill(prompts.cuda())
        eng.set_forced_drafts(cont.cuda(), corrupt.cuda())
        f_log = torch.zeros(max(Kf, W), B, dtype=torch.int32, device="cuda")
        eng.decode_steps(W, None, f_log)
        eng.sync()
        fb = eng.capture(3, (B,), torch.int32).cpu()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        f0.record(eng.stream)
        eng.decode_steps(Kf, None, f_log)
        f1.record(eng.stream)
        eng.sync()
        fa = eng.capture(3, (B,), torch.int32).cpu()
        f_ms, f_tok = dp.reduce_timing(f0.elapsed_time(f1), float(int((fa - fb).sum())), device="cuda")
        f_tok /= tp
        eng.set_forced_drafts(None)
        forced = {"tokens_per_s": f_tok / (f_ms / 1e3), "verify_steps_per_s_per_gpu": Kf / (f_ms / 1e3),
                  "ms_per_step": f_ms / Kf, "mean_accepted_length": f_tok / (Kf * B * world // tp),
                  "a_target": a_target, "alpha": alpha, "steps": Kf,
                  "note": "drafts = GPU greedy continuation corrupted at an i.i.d. slot (seed 2); the draft "
                          "forward still runs every step"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and tp == 1:
        _log("cpu baseline")
        try:
            cpu = oracle_sample(cfg)
        except MemoryError as ex:  # bounded sample did not fit the host
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "strong" if tp > 1 else "weak",
            "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (seeded N(0,0.02) weights, uniform-random prompts)",
            "config": {"workload": f"{cfg.name}-shaped SpecFormer decode step (draft+verify+accept), "
                                   f"batch {B}/GPU, k {k}, prompt {P}",
                       "model": cfg.name, "batch_per_gpu": B if tp == 1 else B / tp, "global_batch": B * world // tp,
                       "draft_len": k, "prompt_len": P, "parallelism": (f"tp{tp}" + ("-fused" if args.tp_fused else "")) if tp > 1 else f"dp{world}",
                       "cuda_graph": True, "logits": "not stored (fused LM-head argmax)" if no_logits else "stored",
                       "l2": "inputs larger than L2 (14 GB weights + KV per step)",
                       "timing": f"median of {n_win} windows of {K} steps, each after a fresh prefill + {W} warm-up steps"},
            "verify_steps_per_s": steps_per_s, "verify_steps_per_s_box": steps_per_s * world,
            "mean_accepted_length": a_meas,
            "forced_acceptance": forced,
            "modeled_tokens_per_s_at_paper_a": steps_per_s * B * world // tp * A_PAPER.get(cfg.name, 1.75),
            "a_paper": A_PAPER.get(cfg.name),
            "roofline": {"bound": ev["bound"], "kernel": dominant, "achieved": ev["achieved"], "peak": ev["peak"],
                         "unit": ev["unit"], "frac": ev["frac"], "traffic": traffic, "peak_source": ev["peak_source"],
                         "algorithmic_units_per_launch": ev["units_per_launch"], "ms_per_launch": ev["ms_per_launch"],
                         "launches_per_step": ev["launches_per_step"],
                         "duration_source": "CUDA event-record nodes around every launch on the engine stream (the "
                                            "step graph re-captured with them; serialises the launches, no PDL "
                                            "overlap), averaged over the profiled steps",
                         "event_classes": ev["classes"], "event_profiled_steps": Kp,
                         "timeline": tl},
            "step_roofline": {"bound": "hbm", "achieved": step_gbs, "peak": hbm, "unit": "GB/s",
                              "frac": step_gbs / hbm, "bytes_per_step": sb / K,
                              "flops_per_step": ev["step_flops"],
                              "t_roof_ms": (sb / K) / (hbm * 1e9) * 1e3},
            "windows": {"n": n_win, "ms": main["all_ms"], "reported": "median"},
            "prefill": prefill,
            "batch_sweep": sweep,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--config", default="7b")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--profile-steps", type=int, default=4)
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = the config's generation length - 1")
    ap.add_argument("--forced-steps", type=int, default=32)
    ap.add_argument("--tp", action="store_true", help="N > 1: split one model over the ranks (tensor parallelism; "
                                                      "the default for --config 70b) instead of one batch per rank")
    ap.add_argument("--tp-fused", action="store_true", help="with --tp: the NEXT-3 fused peer-memory all-reduce "
                    "(CUDA IPC exchange regions) instead of NCCL for the row-parallel outputs")
    ap.add_argument("--timeline-steps", type=int, default=2, help="graph steps replayed with the kernel timeline on")
    ap.add_argument("--draft-len", type=int, default=None, help="override k (13B sweep: 4 / 6 / 8)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--windows", type=int, default=3, help="timed windows (median reported)")
    ap.add_argument("--sweep", default="1,16", help="smaller batches measured in the same run (BASELINE: 1-64)")
    ap.add_argument("--sweep-e2e-steps", type=int, default=64)
    ap.add_argument("--keep-logits", action="store_true", help="store the fp32 logits every step (the API's "
                    "logits read-out; default: not stored, the LM heads' fused argmax gives the tokens)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    args.sweep_list = [int(x) for x in args.sweep.split(",") if x.strip()] if args.sweep not in ("", "none") else []
    from synth import get_config
    cfg = get_config(args.config)
    if args.draft_len is not None:
        cfg = cfg.replace(draft_len=args.draft_len)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
