#!/usr/bin/env python
"""PrefillOnly on B200 — headline benchmark (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl prefillonly|reference]
  (N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...)

Workload (BASELINE.json configs[1]): Llama-3.1-8B bf16, random-init weights, 20,000-token prefill-only
request with a Yes/No allowed list, cold prefix cache. One STEP = one request through the hot path
(hybrid-prefill forward over 32 layers + allowed-row LM head). Request-level data parallelism: every rank
(GPU) runs its own engine on its own requests, no collective on the data path (weak scaling).

  value   prompt tokens/s over the K timed steps, inputs already in HBM (po_prefill_device), device time
          by CUDA events on the engine stream, max over ranks.
  e2e     same metric through the public request API (Engine.prefill: host tokens -> pinned H2D, D2H of
          the allowed-token logits/probs/argmax inside the timed region).
  roofline  per kernel class, algorithmic FLOPs (ps/costs.py:126-136 accounting) / CUDA-event time of
          that class over a second pass of the same K steps (events around every kernel class; kept out of the
          `value` region because they break the PDL overlap); `roofline` is the class with the largest share.
  qps_at_slo  post-recommendation 20k workload (40 users x 50 requests, shared profiles) under Poisson
          arrivals, calibrated SRJF + prefix pool, sticky routing over N GPUs: largest rate whose p99
          latency meets the SLO. Each rank serves its own shard on its own GPU (records gathered for the
          global p99). The event loop is the reference's (serving.simulate, virtual clock); every request of
          the saturation run is executed for real in serving order and its measured device time reused by
          the rate sweep (serving.ReplayServiceFn); a wall-clock Server run at the knee rate is reported beside.
  cpu_baseline  the reference's own layer forward (stock prefillsim block_forward_hybrid from baseline/_ref, numpy
          f64) timed on this host at 1,024 / 2,048 / 4,096 tokens and extrapolated to the 20k request by a fit.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

ALLOWED = [9642, 2822]  # "Yes", "No"
METRIC = "prefill tokens/s (Llama-3.1-8B, 20k-token prefill-only requests)"
UNIT = "tokens/s"
SLO_S = 2.0  # P99 latency SLO for the 20k Llama-8B serving workload (SURVEY §8d proposal, stated)
PEAKS_FALLBACK = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}


def load_peaks() -> tuple[dict, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured (MEASURED_PEAKS.json)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = ROOT / "gpurun_out" / f"clocks_gpu{gpu_index}.csv"

    def __enter__(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self) -> dict:
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, val in zip(names, f[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unsampled"]}
        loaded = [x for x in sm if x > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------------- CPU arm
REF_SIZES = (4096, 8192, 20_000)  # the last is the BASELINE request length: measured, not extrapolated


def _stock_numerics():
    """The reference's own layer forward: prefillsim.numerics from the offline install in baseline/_ref (the stock
    package built from /root/reference, imported unmodified); None when it is not installed."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "prefillsim" / "numerics.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    from prefillsim import numerics

    return numerics


class StockReference:
    """Times the stock reference forward `block_forward_hybrid` (ps/numerics.py:215-275: float64 numpy, chunked
    linear stages, full-length attention) at the Llama-3.1-8B layer shape (hidden 4096, intermediate 14336, chunk
    8192, preallocated in-place outputs) and extrapolates a 20k-token, 32-layer request from a least-squares fit
    t(n) = a*n + b*n^2 over the measured sizes (linear stages ~ n, the reference's full n x n attention ~ n^2)."""

    def __init__(self, numerics, seed: int = 0):
        from paper_2505_07203_b200.config import LLAMA_3_1_8B as M

        self.nm = numerics
        self.M = M
        self.params = numerics.ToyBlockParams.random(seed, M.hidden, M.intermediate)
        self.samples: list[tuple[int, float]] = []

    def step(self, n: int, record: bool = True) -> float:
        x = self.nm.random_input(n, n, self.M.hidden)
        t0 = time.perf_counter()
        self.nm.block_forward_hybrid(self.params, x, 8192, self.nm.ScratchTracker(), prealloc=True, inplace=True)
        dt = time.perf_counter() - t0
        if record:
            self.samples.append((n, dt))
        return dt

    def fit(self) -> tuple[float, float]:
        ns = np.array([n for n, _ in self.samples], dtype=np.float64)
        ts = np.array([t for _, t in self.samples], dtype=np.float64)
        (a, b), *_ = np.linalg.lstsq(np.stack([ns, ns * ns], axis=1), ts, rcond=None)
        return float(a), float(b)

    def request_seconds(self, n_tokens: int) -> float:
        """32 layers x the measured layer time at n_tokens when that length was timed (the fit over small sizes
        underestimated a 20k layer by 1.39x: profiles/r2_reference_fit_check.json), else the fit."""
        at_n = [t for n, t in self.samples if n == n_tokens]
        if at_n:
            return self.M.num_layers * statistics.median(at_n)
        a, b = self.fit()
        return self.M.num_layers * (a * n_tokens + b * n_tokens * n_tokens)

    def summary(self, n_tokens: int) -> dict:
        a, b = self.fit()
        per = {}
        for n, t in self.samples:
            per.setdefault(n, []).append(t)
        return {"layer_seconds": {str(n): statistics.median(v) for n, v in sorted(per.items())},
                "fit_s": {"a_per_token": a, "b_per_token2": b},
                "request_seconds": self.request_seconds(n_tokens),
                "request_from": "32 x measured layer" if any(n == n_tokens for n, _ in self.samples)
                                else "fit extrapolation"}


def cpu_layer_sample(n: int = 1024, seed: int = 0):
    """The CPU port of the path (oracle/llama_ref.py, f64 numpy) on one Llama-8B layer (used when the stock
    reference is not installed, and for the tiny configs[0] request)."""
    from oracle import llama_ref
    from paper_2505_07203_b200.config import LLAMA_3_1_8B as M

    rng = np.random.default_rng(seed)
    h, I, hq, hkv, hd = M.hidden, M.intermediate, M.n_heads, M.n_kv_heads, M.head_dim
    w = lambda r, c: rng.standard_normal((r, c)) / np.sqrt(c)  # noqa: E731
    wq, wk, wv, wo = w(hq * hd, h), w(hkv * hd, h), w(hkv * hd, h), w(h, hq * hd)
    wg, wu, wd = w(I, h), w(I, h), w(h, I)
    x = rng.standard_normal((n, h))
    cfg = llama_ref.Cfg.from_model(M)
    cos, sin = llama_ref.rope_table(cfg, n)
    ones = np.ones(h)

    def run():
        xn = llama_ref.rmsnorm(x, ones, 1e-5, llama_ref._exact)
        q = llama_ref.apply_rope((xn @ wq.T).reshape(n, hq, hd), cos, sin)
        k = llama_ref.apply_rope((xn @ wk.T).reshape(n, hkv, hd), cos, sin)
        v = (xn @ wv.T).reshape(n, hkv, hd)
        y = x + llama_ref.causal_attention(q, k, v).reshape(n, hq * hd) @ wo.T
        xn2 = llama_ref.rmsnorm(y, ones, 1e-5, llama_ref._exact)
        return y + llama_ref.gated_mlp(xn2, wg.T, wu.T, wd.T)

    flops = M.linear_flops_per_token() / M.num_layers * n + M.attn_flops_per_pair() / M.num_layers * n * n / 2
    return run, flops


def tiny_request_seconds() -> float:
    """configs[0]: the tiny 2-layer model's 2,048-token Yes/No request through the CPU oracle (port), seconds."""
    from oracle import llama_ref
    from paper_2505_07203_b200.config import TINY

    cfg = llama_ref.Cfg.from_model(TINY)
    w = llama_ref.make_weights(cfg, 42)
    toks = np.random.default_rng([0, 0, 0]).integers(0, 2 ** 32, size=2048, dtype=np.uint32)
    t0 = time.perf_counter()
    llama_ref.llama_forward(cfg, w, toks, ALLOWED)
    return time.perf_counter() - t0


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"), default=1)
    except Exception:
        return os.cpu_count() or 1


def blas_name() -> str:
    try:
        from threadpoolctl import threadpool_info

        infos = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        return f"{infos[0].get('internal_api')} {infos[0].get('version')}" if infos else "unknown"
    except Exception:
        return "unknown"


def cpu_tokens_per_s(seconds: float, sample_flops: float, n_tokens: int) -> float:
    from paper_2505_07203_b200.config import LLAMA_3_1_8B as M

    rate = sample_flops / seconds  # FLOP/s of the CPU port
    return n_tokens / (M.request_flops(n_tokens) / rate)


def cpu_baseline_sample(n_tokens: int) -> dict:
    """Bounded CPU sample for the GPU arm's `cpu_baseline` (rank 0, N = 1): the stock reference forward at
    REF_SIZES tokens (one layer each, ~10-20 s of CPU work), extrapolated to the request; the port if the
    reference is not installed."""
    nm = _stock_numerics()
    if nm is not None:
        ref = StockReference(nm)
        ref.step(512, record=False)  # warm the BLAS threads
        for n in REF_SIZES:
            ref.step(n)
        sec = ref.request_seconds(n_tokens)
        sm = ref.summary(n_tokens)
        return {"value": n_tokens / sec, "unit": UNIT, "cores": blas_threads(), "kind": "reference",
                "sample": f"stock prefillsim.numerics.block_forward_hybrid (baseline/_ref) at hidden 4096 / "
                          f"intermediate 14336, one layer at each of {list(REF_SIZES)} tokens "
                          f"({', '.join(f'{float(v):.2f} s' for v in sm['layer_seconds'].values())}); request = "
                          f"{sm['request_from']} ({n_tokens} tokens, 32 layers)",
                "fit": sm, "blas": blas_name(), "host_cpus": os.cpu_count()}
    run, flops = cpu_layer_sample()
    run()
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < 10.0 or reps < 2:
        run()
        reps += 1
    sec = (time.perf_counter() - t0) / reps
    return {"value": cpu_tokens_per_s(sec, flops, n_tokens), "unit": UNIT, "cores": blas_threads(), "kind": "port",
            "sample": f"{reps} x one Llama-3.1-8B layer at 1,024 tokens (float64 numpy CPU port of the reference "
                      f"path, oracle/llama_ref.py), {sec:.2f} s each, extrapolated by the FLOP formula to 32 layers "
                      f"x {n_tokens} tokens", "host_cpus": os.cpu_count()}


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU implementation of the path on the host cores.

    Each step runs the stock `prefillsim.numerics.block_forward_hybrid` (installed unmodified into baseline/_ref)
    for one Llama-8B-shaped layer at 1,024 / 2,048 / 4,096 tokens in turn; the value is the 20k-token, 32-layer
    request extrapolated from the fit over all timed steps. The CPU port (oracle/llama_ref.py) is the fallback
    when the install is missing."""
    if rank != 0:
        return
    # every host thread for the BLAS (torchrun sets OMP_NUM_THREADS=1 for its workers; the other ranks idle here)
    try:
        from threadpoolctl import threadpool_limits

        limits = threadpool_limits(limits=os.cpu_count() or 1, user_api="blas")
    except Exception:
        limits = None
    nm = _stock_numerics()
    extra = {}
    if nm is not None:
        ref = StockReference(nm)
        for i in range(args.warmup):
            ref.step(REF_SIZES[0], record=False)
        t_all = 0.0
        for i in range(args.steps):
            t_all += ref.step(REF_SIZES[i % len(REF_SIZES)])
        if not any(n == args.n_tokens for n, _ in ref.samples):  # the request length itself is always timed
            t_all += ref.step(args.n_tokens)
        if len({n for n, _ in ref.samples}) < 2:  # the reported fit needs two sizes
            t_all += ref.step(REF_SIZES[0])
        request_s = ref.request_seconds(args.n_tokens)
        value = args.n_tokens / request_s
        kind = "reference"
        sample = (f"stock prefillsim.numerics.block_forward_hybrid (baseline/_ref, unmodified) at hidden 4096 / "
                  f"intermediate 14336, one layer per step cycling {list(REF_SIZES)} tokens; request = 32 x the "
                  f"measured {args.n_tokens}-token layer ({request_s:.0f} s per request)")
        extra = {"fit": ref.summary(args.n_tokens)}
        ms_per_step = 1e3 * t_all / max(1, len(ref.samples))
    else:
        run, flops = cpu_layer_sample()
        for _ in range(args.warmup):
            run()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            run()
            times.append(time.perf_counter() - t0)
        value = cpu_tokens_per_s(sum(times) / args.steps, flops, args.n_tokens)
        kind = "port"
        sample = (f"one Llama-3.1-8B layer at 1,024 tokens in float64 numpy per step (oracle/llama_ref.py), "
                  f"extrapolated by the FLOP formula to 32 layers x {args.n_tokens} tokens")
        ms_per_step = 1e3 * sum(times) / args.steps
    try:
        extra["tiny_config0_request_s"] = tiny_request_seconds()
    except Exception as exc:  # noqa: BLE001 - informational only
        extra["tiny_config0_request_s"] = f"failed: {exc}"
    cores = blas_threads()
    if limits is not None:
        limits.restore_original_limits()
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (random weights, random activations)",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                         "blas": blas_name(), "host_cpus": os.cpu_count(), **extra},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference (arxiv 2505.07203 prefillsim) models serving analytically; its own implementation of "
                "the layer forward (ps/numerics.py block_forward_hybrid, single-head toy block, float64) is what "
                "runs here. tiny_config0_request_s: BASELINE configs[0] through the CPU port oracle",
    }), flush=True)


def workload_config(args, world) -> dict:
    return {"workload": f"Llama-3.1-8B bf16 random-init, {args.n_tokens}-token prefill-only request, Yes/No "
                        "allowed ids, cold prefix cache (BASELINE configs[1])",
            "model": "llama-3.1-8b", "n_tokens": args.n_tokens, "global_batch": world, "seq_len": args.n_tokens,
            "chunk": args.chunk, "parallelism": f"dp{world} (request-level, no data-path collective)",
            "l2": "inputs larger than L2: 16 GB of weights stream through a 126 MB L2 every step"}


# ---------------------------------------------------------------------------------------------- GPU arm
def executed_flops_per_class(M, n: int, last_row_only: bool) -> dict:
    """Executed FLOPs per kernel class for one cold n-token request (the last layer runs attention, O and
    the MLP for the final row only when last_row_only)."""
    h, I = M.hidden, M.intermediate
    qkvc = (M.n_heads + 2 * M.n_kv_heads) * M.head_dim
    ctx = M.n_heads * M.head_dim
    L = M.num_layers
    rows = (L - 1) * n + 1 if last_row_only else L * n  # row-layers through attention output / O / MLP
    pairs = (L - 1) * n * n / 2.0 + n if last_row_only else L * n * n / 2.0
    # MLP: layers whose MLP rows exceed 256 run the fused gate/up + down launch (mlp_fused, when enabled); the last
    # layer's single row (last_row_only) runs the separate GEMMs
    fused_rows = ((L - 1) * n if last_row_only else L * n) if n > 256 else 0
    sep_rows = rows - fused_rows
    return {"gemm_qkv_rope": 2.0 * n * h * qkvc * L, "gemm_o_resid": 2.0 * rows * ctx * h,
            "gemm_gate_up_silu": 2.0 * sep_rows * h * 2 * I, "gemm_down_resid": 2.0 * sep_rows * I * h,
            "mlp_fused": 2.0 * fused_rows * h * 3 * I,
            "gemm_gate_up_silu_if_separate": 2.0 * rows * h * 2 * I, "gemm_down_resid_if_separate": 2.0 * rows * I * h,
            "attention": 4.0 * h * pairs}


def hbm_bytes_per_class(M, n: int, n_allowed: int) -> dict:
    """Algorithmic DRAM bytes per request of the memory-bound kernel classes (cold n-token request)."""
    h = M.hidden
    # embedding rows (bf16) in; fp32 residual, bf16 folded-norm input and per-128-column sums of squares out
    embed = n * h * 2 + n * h * 4 + n * h * 2 + n * (h // 128) * 4
    # last residual row + final norm gamma + the allowed LM-head rows in; logits / probs / argmax out
    lm_head = h * 4 + h * 4 + n_allowed * h * 2 + n_allowed * 8 + 4
    return {"embed": embed, "lm_head": lm_head}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="prefillonly", choices=["prefillonly", "reference", "ours"])
    ap.add_argument("--n-tokens", type=int, default=20_000)
    ap.add_argument("--chunk", type=int, default=8192)
    ap.add_argument("--no-qps", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slo", type=float, default=SLO_S)
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import torch.distributed as dist

    from paper_2505_07203_b200.config import LLAMA_3_1_8B as M
    from paper_2505_07203_b200.engine import Engine

    ndev = torch.cuda.device_count()
    local = local % ndev  # one process per GPU; more ranks than GPUs only in single-GPU validation runs
    torch.cuda.set_device(local)
    if world > 1:
        # control plane only (barrier + max-over-ranks timing): no collective touches the data path
        if ndev >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    n = args.n_tokens
    K, W = args.steps, args.warmup
    eng = Engine(M, device=local, seed=0, max_tokens=max(n, 24_000), chunk=args.chunk, pool_blocks=24_576)
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))

    # distinct synthetic requests per step and rank, resident in HBM before the timed region
    reqs = [np.random.default_rng([rank, 1, i]).integers(0, 2 ** 32, size=n, dtype=np.uint32) for i in range(K + W)]
    d_tok = [torch.from_numpy(r.view(np.int32)).to(f"cuda:{local}") for r in reqs]
    d_allowed = torch.tensor(ALLOWED, dtype=torch.int32, device=f"cuda:{local}")
    d_logits = torch.empty(len(ALLOWED), dtype=torch.float32, device=f"cuda:{local}")
    d_probs = torch.empty_like(d_logits)
    d_argmax = torch.empty(1, dtype=torch.int32, device=f"cuda:{local}")
    torch.cuda.synchronize()

    def step(i):
        eng.prefill_device(d_tok[i].data_ptr(), n, d_allowed.data_ptr(), len(ALLOWED), d_logits.data_ptr(),
                           d_probs.data_ptr(), d_argmax.data_ptr())

    for i in range(W):
        step(K + i)
    torch.cuda.synchronize()
    launches_per_step = eng.last_launches

    # ---------------- timed region: value (device time, inputs resident)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(K):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    elapsed_ms = max_over_ranks(ev0.elapsed_time(ev1))
    value = world * K * n / (elapsed_ms / 1e3)
    clocks = clk.summary()

    # ---------------- the same K steps again with CUDA events around every kernel class (live per-kernel timing
    # for the roofline; kept out of the timed region above because events between kernels break the PDL overlap)
    barrier()
    torch.cuda.synchronize()
    eng.profile_begin()
    for i in range(K):
        step(i)
    torch.cuda.synchronize()
    prof = eng.profile_end()
    barrier()

    # ---------------- e2e through the public API (host tokens, H2D + D2H inside the region)
    results = []
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(K):
        results.append(eng.prefill(reqs[i], ALLOWED))
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    barrier()
    e2e = {"value": world * K * n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": n * 4 + 4 * len(ALLOWED),
           "d2h_bytes_per_step": 8 * len(ALLOWED) + 4,
           "note": "Engine.prefill: pinned-staged H2D of the token ids, forward, D2H of logits/probs/argmax; "
                   "wall clock, max over ranks"}

    # ---------------- roofline per kernel class (algorithmic FLOPs / CUDA-event time in the timed region)
    peaks, peak_src = load_peaks()
    sustained = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    cls_flops = executed_flops_per_class(M, n, eng.last_row_only)
    cls_bytes = hbm_bytes_per_class(M, n, len(ALLOWED))
    total_ms = sum(v[0] for v in prof.values())
    traffic = {}
    tpath = ROOT / "profiles" / "ncu_traffic.json"
    if tpath.exists():
        traffic = json.loads(tpath.read_text()).get("dram_bytes_per_launch", {})
    by_kernel = {}
    if prof.get("mlp_fused", (0, 0))[1] == 0:  # per-chunk MLP launches (PO_FUSED_MLP=0): all MLP rows separate
        cls_flops["gemm_gate_up_silu"] = cls_flops["gemm_gate_up_silu_if_separate"]
        cls_flops["gemm_down_resid"] = cls_flops["gemm_down_resid_if_separate"]
    for name, (ms, cnt) in prof.items():
        if cnt == 0:
            continue  # kernel classes this forward does not launch (norm folded into GEMMs, gather in A/B mode only)
        entry = {"ms_per_step": ms / K, "launches_per_step": cnt / K, "share": ms / total_ms if total_ms else 0.0}
        if name in cls_flops and ms > 0:
            ach = cls_flops[name] * K / (ms / 1e3) / 1e12
            entry.update({"bound": "tensor", "achieved": ach, "unit": "TFLOP/s", "peak": sustained,
                          "frac": ach / sustained, "frac_of_burst": ach / peaks["bf16_tflops"]})
        elif name in cls_bytes and ms > 0:
            gbs = cls_bytes[name] * K / (ms / 1e3) / 1e9
            entry.update({"bound": "hbm" if name != "lm_head" else "latency", "achieved": gbs, "unit": "GB/s",
                          "peak": peaks["hbm_gbs"], "frac": gbs / peaks["hbm_gbs"],
                          "bytes_per_request": cls_bytes[name]})
        by_kernel[name] = entry
    top = max((k for k in by_kernel if by_kernel[k].get("unit") == "TFLOP/s"), key=lambda k: by_kernel[k]["share"])
    t = by_kernel[top]
    roofline = {"kernel": top, "bound": "tensor", "achieved": t["achieved"], "peak": sustained, "unit": "TFLOP/s",
                "frac": t["frac"], "traffic": traffic.get(top),
                "peak_source": f"{peak_src}: bf16_tflops_sustained (kernel timed inside a long step); "
                               f"burst {peaks['bf16_tflops']} gives frac {t['frac_of_burst']:.3f}",
                "per_launch": f"{cls_flops[top] / max(1, prof[top][1] // K):.4g} algorithmic FLOP per launch"}
    from paper_2505_07203_b200.config import executed_flops

    whole = M.request_flops(n) * world * K / (elapsed_ms / 1e3) / 1e12
    exe = executed_flops(M, n, 0, eng.last_row_only)
    whole_exe = exe * world * K / (elapsed_ms / 1e3) / 1e12
    step_roofline = {"achieved": whole, "unit": "TFLOP/s", "frac": whole / world / sustained,
                     "frac_of_burst": whole / world / peaks["bf16_tflops"],
                     "flops_per_request": M.request_flops(n),
                     "executed_flops_per_request": exe, "achieved_executed": whole_exe,
                     "frac_executed": whole_exe / world / sustained,
                     "note": "algorithmic = reference accounting (ps/costs.py:126-136,275-277); executed skips the "
                             "last layer's attention/O/MLP for rows other than the final one (exact)"}

    # ---------------- QPS at P99 SLO (calibrated SRJF + prefix pool, DP over all ranks)
    qps = None
    if not args.no_qps:
        qps = qps_at_slo(eng, M, world, rank, args.slo, dist if world > 1 else None)
        barrier()

    # ---------------- prefix-hit forward (the serving path after a cache hit): an HBM-bound weight stream
    hit = prefix_hit_roofline(eng, M, n, peaks) if rank == 0 and not args.no_qps else None

    # ---------------- CPU baseline (rank 0, N = 1 only): the stock reference forward on a bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(n)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": elapsed_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (counter-hash random-init weights, seeded uint32 token streams)",
            "config": workload_config(args, world), "e2e": e2e, "gpu_launches": launches_per_step * K,
            "roofline": roofline, "roofline_by_kernel": by_kernel, "step_roofline": step_roofline,
            "cpu_baseline": cpu, "qps_at_slo": qps, "prefix_hit": hit, "clocks": clocks,
            "answer": {"argmax": results[-1].token, "probs": results[-1].probs.tolist()},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def prefix_hit_roofline(eng, M, n, peaks):
    """A warm prefix-hit request (all but the last 160 tokens cached, block-aligned) measured back to back: device
    service time and its HBM roofline. One hit streams every layer weight once plus the cached K/V of all layers
    (read by attention straight from the pool), so its floor is those bytes at the measured copy bandwidth."""
    toks = np.random.default_rng([7, 1, 0]).integers(0, 2 ** 32, size=n, dtype=np.uint32)
    nb = n // 16
    slots = list(range(nb))
    eng.prefill(toks, ALLOWED, 0, slots)  # admit the prefix
    nc = (n - 160) // 16 * 16
    for _ in range(5):  # back-to-back hits settle the clocks after the cold forward
        eng.prefill(toks, ALLOWED, nc, slots)
    ts = sorted(eng.prefill(toks, ALLOWED, nc, slots).service_s for _ in range(15))
    med = ts[len(ts) // 2]
    # where a hit's time goes: CUDA events around every kernel class over 10 more hits (events break the PDL overlap,
    # so the classes sum to more than the plain service time: compare shares)
    eng.profile_begin()
    for _ in range(10):
        eng.prefill(toks, ALLOWED, nc, slots)
    prof = eng.profile_end()
    per_class = {k: {"ms_per_hit": ms / 10, "launches_per_hit": cnt // 10} for k, (ms, cnt) in prof.items() if cnt}
    lin_weights = M.weight_bytes - 2 * (2 * M.vocab * M.hidden)  # embedding / LM head rows are gathered, not streamed
    kv = M.kv_bytes_per_token[1] * n
    bytes_ = lin_weights + kv
    achieved = bytes_ / med / 1e9
    return {"n": n, "n_cached": nc, "service_ms_median": med * 1e3, "service_ms_min": ts[0] * 1e3,
            "bytes_per_request": bytes_, "achieved_gbs": achieved, "peak_gbs": peaks["hbm_gbs"],
            "frac": achieved / peaks["hbm_gbs"], "bound": "hbm", "per_class_events": per_class,
            "note": "algorithmic bytes = layer weights streamed once + cached K/V of all layers read once; "
                    "back-to-back hits (inside a mixed serving run the clocks are still recovering from cold "
                    "forwards: see qps_at_slo.measured_service_s.prefix_hit_median)"}


def qps_at_slo(eng, M, world, rank, slo, dist):
    """Calibrated-SRJF serving of the post-recommendation 20k workload, request-level DP over `world` GPUs.

    Every rank serves its own shard of the trace (sticky user routing, `serving.shard_trace`, ps/sim.py:52-66) on its
    own engine and prefix pool; the per-rank records are gathered (`merge_records`) for the global p99, and every
    rank takes the same decisions from the merged report. Virtual-clock event loop with the reference's semantics
    (serving.simulate, ps/sim.py:211-269): each rank's requests of the saturation run execute for real on that
    rank's GPU in serving order (ReplayServiceFn) and the rate sweep reuses those device times. At the knee rate a
    wall-clock run (serving.Server + replay: real arrivals in real time, host-side hashing, scheduling and ctypes
    inside the latency) is reported beside it.
    """
    from paper_2505_07203_b200 import jct as J
    from paper_2505_07203_b200 import workload as wl
    from paper_2505_07203_b200.scheduling import SCORING_PROFILE, Policy
    from paper_2505_07203_b200.serving import (ReplayServiceFn, Server, merge_records, qps_at_slo as pick,
                                               refine_qps, replay, shard_trace, simulate, sweep_rates)

    trace = wl.gen_post_recommendation(0, wl.POSTREC_20K)
    capacity = min(eng.capacity_tokens, 16 * eng.pool_blocks)
    t0 = time.perf_counter()

    def merged(local):
        if world == 1:
            return local
        allr = [None] * world
        dist.all_gather_object(allr, list(local.records))
        return merge_records(allr, world)

    # the paper's calibration: JCT profile fitted on this GPU's measured latencies
    # (ps/jct.py:100-128 with the real engine as latency_fn), seconds-valued scores, lambda = 500
    jprof = J.fit(J.profile_engine(eng, max_input=24_000, step=4000))
    svc = ReplayServiceFn(eng, ALLOWED)

    def run(tr, pol=None, jp=None):
        mine = shard_trace(tr, rank, world)
        return merged(simulate(mine, 1, pol or Policy.srjf_calibrated(), capacity, svc, jct_profile=jp))

    sat_rep = run(wl.zero_arrivals(trace))  # every request runs for real here, in its rank's serving order
    sat = sat_rep.throughput
    svc.recording = False
    rates = [sat * m for m in (0.25, 0.5, 0.75, 0.9, 1.0, 1.1, 1.25, 1.5, 2.0)]
    sweep = lambda pol, jp=None: (lambda tr: run(tr, pol, jp))  # noqa: E731
    res = sweep_rates(trace, rates, seed=0, run=sweep(None))
    fifo = sweep_rates(trace, rates, seed=0, run=sweep(Policy.fifo()))
    # resolve the knee: bisect between the last rate meeting the SLO and the first one above it that misses
    res = refine_qps(res, slo, lambda q: sweep_rates(trace, [q], seed=0, run=sweep(None))[0][1])
    fifo = refine_qps(fifo, slo, lambda q: sweep_rates(trace, [q], seed=0, run=sweep(Policy.fifo()))[0][1])
    polp = Policy.srjf_calibrated(lam=500.0, scoring=SCORING_PROFILE)
    resp = refine_qps(sweep_rates(trace, rates, seed=0, run=sweep(polp, jprof)), slo,
                      lambda q: sweep_rates(trace, [q], seed=0, run=sweep(polp, jprof))[0][1])
    best = pick(res, slo)
    rep = dict(res)[best] if best else None
    # lambda sweep at one rate past the knee (the reference's `lambda-sweep`, ps/cli.py:213-252): the fairness
    # weight trades mean latency (SRJF) against the p99 of the long cold requests (FIFO)
    lam_rate = 1.1 * best if best else sat
    arrived = wl.poisson_arrivals(trace, lam_rate, seed=0, keep_sessions=True)
    lam_sweep = []
    for lam in (0.0, 0.5, 5.0, 50.0, 500.0, 5000.0):
        r = run(arrived, Policy.srjf_calibrated(lam=lam))
        lam_sweep.append({"lambda": lam, "scoring": "proxy (miss tokens)", "p99_s": r.p99_latency,
                          "mean_s": r.mean_latency})
    for lam in (0.0, 0.5, 500.0):
        r = run(arrived, Policy.srjf_calibrated(lam=lam, scoring=SCORING_PROFILE), jprof)
        lam_sweep.append({"lambda": lam, "scoring": "profile (seconds)", "p99_s": r.p99_latency,
                          "mean_s": r.mean_latency})
    rf = run(arrived, Policy.fifo())
    lam_sweep.append({"policy": "fifo", "p99_s": rf.p99_latency, "mean_s": rf.mean_latency})
    # wall clock: serving.Server (lookahead loop, C-ABI forwards, host-side hashing / scheduling / copies inside the
    # latency) with real arrivals in real time. First its saturation throughput (every request at t = 0), then the
    # highest of {1.0, 0.95, 0.9, 0.85, 0.8} x the virtual-clock knee whose wall-clock p99 meets the SLO, refined by
    # three bisection steps toward the next grid rate that misses it.
    wall = None
    if best:
        def wall_run(tr):
            if world > 1:
                dist.barrier()
            srv = Server([eng], Policy.srjf_calibrated())
            try:
                return merged(replay(srv, shard_trace(tr, rank, world), ALLOWED))
            finally:
                srv.close()

        wsat = wall_run(wl.zero_arrivals(trace))
        runs = []
        for m in (1.0, 0.95, 0.9, 0.85, 0.8):
            q = best * m
            wrep = wall_run(wl.poisson_arrivals(trace, q, seed=0, keep_sessions=True))
            runs.append({"rate": q, "p99_s": wrep.p99_latency, "mean_s": wrep.mean_latency,
                         "throughput_rps": wrep.throughput, "served": wrep.served})
            if wrep.p99_latency <= slo:
                break
        # resolve the wall-clock knee below the grid's 5% steps: bisect between the passing rate and the failing one
        passing = [r["rate"] for r in runs if r["p99_s"] <= slo]
        failing = [r["rate"] for r in runs if r["p99_s"] > slo]
        if passing and failing:
            lo, hi = max(passing), min(f for f in failing if f > max(passing))
            for _ in range(3):
                q = 0.5 * (lo + hi)
                wrep = wall_run(wl.poisson_arrivals(trace, q, seed=0, keep_sessions=True))
                runs.append({"rate": q, "p99_s": wrep.p99_latency, "mean_s": wrep.mean_latency,
                             "throughput_rps": wrep.throughput, "served": wrep.served})
                if wrep.p99_latency <= slo:
                    lo = q
                else:
                    hi = q
        ok = [r["rate"] for r in runs if r["p99_s"] <= slo]
        wall = {"qps_at_slo": max(ok) if ok else None, "saturation_rps": wsat.throughput,
                "virtual_saturation_rps": sat, "runs": runs,
                "note": "serving.Server (lookahead: next decision while the current forward runs) + replay: arrivals "
                        "injected in real time, wall-clock latency incl. host hashing, scheduling, staging copies"}
    hits = sorted(v[0] for (rid, nc), v in svc.by_request.items() if nc > 0)
    colds = sorted(v[0] for (rid, nc), v in svc.by_request.items() if nc == 0)
    if rank != 0:
        return None
    return {
        "value": best, "unit": "requests/s", "slo_p99_s": slo, "n_gpus": world,
        "prompt_tokens_per_s_at_slo": rep.prompt_tokens_per_s if rep else None,
        "miss_tokens_per_s_at_slo": rep.miss_tokens_per_s if rep else None,
        "p99_at_value_s": rep.p99_latency if rep else None,
        "fifo_qps_at_slo": pick(fifo, slo),
        "profile_lambda500_qps_at_slo": pick(resp, slo),
        "wall_clock": wall,
        "lambda_sweep": {"rate": lam_rate, "runs": lam_sweep},
        "jct_profile": {"coef_input": jprof.coef_input, "coef_cached": jprof.coef_cached,
                        "intercept": jprof.intercept, "fit_r2": jprof.fit_r2},
        "saturation_rps": sat,
        "sweep": [{"rate": q, "p99_s": r.p99_latency, "mean_s": r.mean_latency, "hit_requests": r.cache_hit_requests}
                  for q, r in res],
        "fifo_sweep": [{"rate": q, "p99_s": f.p99_latency} for q, f in fifo],
        "search": "grid of 0.25-2.0 x the saturation rate, then 5 bisection steps between the last rate meeting the "
                  "SLO and the next one missing it",
        "workload": "post-recommendation 40 users x 50 requests, profiles 19,850 +- 3,000 tokens + 150-token "
                    "suffix, Poisson arrivals (user sessions contiguous), Yes/No allowed ids",
        "method": f"virtual-clock serving loop with the reference's event semantics (calibrated SRJF, prefix pool of "
                  f"{capacity} tokens per GPU); each of the {world} rank(s) serves its sticky-routed shard on its own "
                  f"GPU (saturation run executed for real in serving order, device times reused by the rate sweep; "
                  f"shapes beyond those: one forward each), records merged over ranks; rank 0: {svc.forwards} real "
                  f"forwards ({time.perf_counter() - t0:.1f} s wall)",
        "measured_service_s": {"cold_median": statistics.median(colds) if colds else None,
                               "prefix_hit_median": statistics.median(hits) if hits else None},
    }


if __name__ == "__main__":
    main()
