"""Benchmark driver (contract in the task statement; workload = BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload bert|c1]

Default workload: BERT-base full INT8 W8A8 encoder forward, batch 32 x seq 128,
random-init weights (Gaussian 0.02), synthetic token ids, 12 post-LN blocks
(reference transformer.py:443-486) + final LN; metric = sequences / second.
A step = one forward of the whole batch.  Multi-GPU: one process per GPU, each
rank runs its own replica of the batch (the encoder does not shard: "replicas
only"), value = all ranks' sequences / max-over-ranks time.

Timing: W warm-up steps, then K steps, each bracketed by CUDA events on the
launching stream with an L2 flush (256 MiB memset) between steps outside the
events; barrier + synchronize on both sides; max over ranks.

--impl reference: the reference algorithm on the host CPU (the oracle port of
lowbit's numpy path with its int64 igemm), all host cores via a process pool,
bounded sample: one block on one sequence per core per step, extrapolated to
the full 12-layer forward.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BERT = dict(layers=12, hidden=768, heads=12, ffn=3072, batch=32, seq=128, groups=48, vocab=30522)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ---------------------------------------------------------------------------
# CPU reference arm / baseline
# ---------------------------------------------------------------------------


def _ref_layer_worker(seed: int) -> float:
    """One post-LN block forward of one 128-token BERT-base sequence with the
    reference algorithm (oracle restatement, int64 igemm as igemm.py:79)."""
    import numpy as np

    from oracle import lowbit_oracle as O

    O.use_reference_cost_igemm(True)
    d, f, heads, seq = BERT["hidden"], BERT["ffn"], BERT["heads"], BERT["seq"]
    rng = O.Rng(seed)
    w = {n: rng.gaussian(s, std=0.02) for n, s in (
        ("w_q", (d, d)), ("w_k", (d, d)), ("w_v", (d, d)), ("w_o", (d, d)),
        ("w_h4h", (f, d)), ("w_4hh", (d, f)))}
    for n, s in (("b_q", d), ("b_k", d), ("b_v", d), ("b_o", d), ("b_h4h", f), ("b_4hh", d),
                 ("ln1_beta", d), ("ln2_beta", d)):
        w[n] = np.zeros(s, np.float32)
    w["ln1_gamma"] = np.ones(d, np.float32)
    w["ln2_gamma"] = np.ones(d, np.float32)
    qb = O.quantize_block(w, 8, 8, BERT["groups"])
    x = O.Rng(seed + 1).gaussian((seq, d), std=0.5)
    t0 = time.perf_counter()
    O.block_forward(x, qb, heads, False, "int8")
    return time.perf_counter() - t0


class RefPool:
    """Process pool running the reference block forward, one sequence per core."""

    def __init__(self, cores: int):
        from concurrent.futures import ProcessPoolExecutor

        self.cores = cores
        self.ex = ProcessPoolExecutor(max_workers=cores)
        list(self.ex.map(_ref_layer_worker, range(cores)))  # warm (imports, page-in)
        self.r = 0

    def round(self) -> float:
        self.r += 1
        t0 = time.perf_counter()
        list(self.ex.map(_ref_layer_worker, range(100 * self.r, 100 * self.r + self.cores)))
        return time.perf_counter() - t0

    def close(self):
        self.ex.shutdown()


def cpu_reference_sample(cores: int, rounds: int = 1, pool: "RefPool | None" = None):
    """Returns (seq/s for the full 12-layer forward, sample description, wall s)."""
    own = pool is None
    pool = pool or RefPool(cores)
    walls = [pool.round() for _ in range(rounds)]
    if own:
        pool.close()
    wall = statistics.median(walls)
    seq_per_s = cores / (wall * BERT["layers"])
    sample = (f"{cores} process(es) x 1 post-LN block x 1 sequence of {BERT['seq']} tokens "
              f"(BERT-base W8A8, reference numpy algorithm with int64 igemm), median of {rounds}; "
              f"extrapolated x{BERT['layers']} layers")
    return seq_per_s, sample, wall


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    pool = RefPool(cores)
    for _ in range(args.warmup):
        pool.round()
    vals = []
    for _ in range(args.steps):
        v, sample, _ = cpu_reference_sample(cores, 1, pool)
        vals.append(v)
    pool.close()
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "BERT-base W8A8 encoder forward throughput", "value": value,
        "unit": "seq/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * BERT["batch"] / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int8", "data": "synthetic",
        "config": workload_config(),
        "cpu_baseline": {"value": value, "unit": "seq/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "seq/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def workload_config():
    return {"workload": "BERT-base full INT8 W8A8 encoder forward (BASELINE configs[1])",
            "global_batch": BERT["batch"], "seq_len": BERT["seq"], "layers": BERT["layers"],
            "hidden": BERT["hidden"], "heads": BERT["heads"], "ffn": BERT["ffn"],
            "weight_groups": BERT["groups"], "activations": "dynamic token-wise int8",
            "attention": "fp32", "parallelism": "replicas", "l2": "flushed (256 MiB memset) between timed steps"}


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def build_engine(torch, seed_base: int = 0):
    from paper_2206_01861_b200 import transformer as T

    blocks = [T.random_block(BERT["hidden"], BERT["heads"], 8, 8, BERT["groups"], seed=seed_base + i,
                             ffn_mult=BERT["ffn"] // BERT["hidden"]) for i in range(BERT["layers"])]
    gen = torch.Generator(device="cuda").manual_seed(seed_base + 999)
    emb = torch.randn((BERT["vocab"], BERT["hidden"]), generator=gen, device="cuda") * T.INIT_STD
    eng = T.EncoderEngine(blocks=blocks, embedding=emb, final_gamma=torch.ones(BERT["hidden"], device="cuda"),
                          final_beta=torch.zeros(BERT["hidden"], device="cuda"), batch=BERT["batch"],
                          seq=BERT["seq"], causal=False)
    return eng


def gemm_roofline(torch, eng, peaks, basis):
    """Time every fused W8A8 linear of one eager forward with CUDA events on the
    launching stream; achieved = algorithmic ops / summed launch time."""
    from paper_2206_01861_b200 import _native as N

    events = []
    orig = eng._linear

    def timed_linear(q, s, w, bias, out):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        orig(q, s, w, bias, out)
        b.record()
        events.append((a, b, 2 * q.shape[0] * q.shape[1] * w.rows))

    eng._linear = timed_linear
    try:
        for _ in range(3):
            events.clear()
            eng._run()
        torch.cuda.synchronize()
    finally:
        eng._linear = orig
    t = sum(a.elapsed_time(b) * 1e-3 for a, b, _ in events)
    ops = sum(o for _, _, o in events)
    achieved = ops / t / 1e12
    peak = 2.0 * peaks["bf16_tflops"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("bert_gemm_bytes_per_launch")
    _ = N
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": "zq_gemm_kernel (fused W8A8 linear, tcgen05 kind::i8)",
            "launches_per_step": len(events),
            "peak_basis": f"2 x {basis} bf16 dense ({peaks['bf16_tflops']} TF/s, MEASURED_PEAKS.json): "
                          "kind::i8 issues at twice the kind::f16 rate",
            "per_launch_us": 1e6 * t / max(1, len(events))}


def run_ours(args, rank: int, world: int, dist):
    import numpy as np
    import torch

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    peaks, basis = load_peaks()
    eng = build_engine(torch, seed_base=0)
    eng.capture()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    ids_host = torch.from_numpy(np.random.default_rng(rank).integers(0, BERT["vocab"], (BERT["batch"], BERT["seq"]))
                                ).pin_memory()
    eng._bufs["ids"].copy_(ids_host.reshape(-1).cuda())
    for _ in range(args.warmup):
        eng.launch()
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident throughput (value) ----
    stream = torch.cuda.current_stream()
    times = []
    barrier()
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            eng.launch()
            b.record(stream)
            times.append((a, b))
        barrier()
    step_s = [a.elapsed_time(b) * 1e-3 for a, b in times]
    total = sum(step_s)
    eng.check_finite()

    # ---- end to end through the public API with host buffers ----
    out_host = torch.empty((eng.tokens, BERT["hidden"]), dtype=torch.float32).pin_memory()
    e2e_times = []
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = eng.forward(ids_host)          # H2D of ids inside
        out_host.copy_(out, non_blocking=True)  # D2H of the result
        b.record(stream)
        e2e_times.append((a, b))
    barrier()
    e2e_total = sum(a.elapsed_time(b) * 1e-3 for a, b in e2e_times)

    if dist is not None:
        t = torch.tensor([total, e2e_total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total, e2e_total = float(t[0]), float(t[1])

    seqs = BERT["batch"] * world * args.steps
    value = seqs / total
    e2e_value = seqs / e2e_total
    roof = gemm_roofline(torch, eng, peaks, basis) if rank == 0 else None
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    cpu_val, cpu_sample, _ = cpu_reference_sample(cores, 1)
    launches_per_step = 2 + 8 * BERT["layers"]
    line = {
        "metric": "BERT-base W8A8 encoder forward throughput", "value": value, "unit": "seq/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int8", "data": "synthetic (random-init weights, random token ids)",
        "config": workload_config(),
        "e2e": {"value": e2e_value, "unit": "seq/s", "h2d_bytes_per_step": int(ids_host.numel() * 8),
                "d2h_bytes_per_step": int(out_host.numel() * 4)},
        "roofline": roof,
        "cpu_baseline": {"value": cpu_val, "unit": "seq/s", "cores": cores, "kind": "port", "sample": cpu_sample},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
        "step_ms_min_max": [1000 * min(step_s), 1000 * max(step_s)],
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl")
        dist = tdist
    run_ours(args, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
