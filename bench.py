"""Benchmark driver (contract in the task statement; workload = BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload all|bert|c1|c1-f16|gemm-large|wo-gemm|gpt3-350m|gptj-6b|neox-20b]

Headline workload (the JSON line's metric/value): BERT-base full INT8 W8A8
encoder forward, batch 32 x seq 128, random-init weights (Gaussian 0.02),
synthetic token ids, 12 post-LN blocks (reference transformer.py:443-486) +
final LN; metric = sequences / second.  A step = one forward of the whole
batch.  Multi-GPU: one process per GPU, each rank runs its own replica of the
batch (the encoder does not shard: "replicas only"), value = all ranks'
sequences / max-over-ranks time.

With the default `--workload all` the same line also carries, under
"workloads", the other BASELINE configurations measured in the same run (each
with its own value / unit / e2e / roofline): configs[0] (C1 quantized linear,
f32 and fp16 out), large-shape W8A8 GEMMs (TOPS vs the INT8 peak), and the GPT
generation workloads (configs[2-4]); the GPT models run Megatron tensor
parallel over all N ranks (GPT-NeoX 20B at TP = N is the metric's
"tok/s 1-8 GPU" clause).  `--workload X` prints X's own line instead.

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
        "extrapolated": True,
        "extrapolation": f"each step times {cores} one-block, one-sequence reference forwards in parallel and "
                         f"scales the wall time x{BERT['layers']} layers to the 12-layer forward; ms_per_step is "
                         f"that estimate per {BERT['batch']}-sequence batch, not a measured wall time",
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


def build_engine(torch, seed_base: int = 0, lanes: int | None = None):
    from paper_2206_01861_b200 import transformer as T

    blocks = [T.random_block(BERT["hidden"], BERT["heads"], 8, 8, BERT["groups"], seed=seed_base + i,
                             ffn_mult=BERT["ffn"] // BERT["hidden"]) for i in range(BERT["layers"])]
    gen = torch.Generator(device="cuda").manual_seed(seed_base + 999)
    emb = torch.randn((BERT["vocab"], BERT["hidden"]), generator=gen, device="cuda") * T.INIT_STD
    eng = T.EncoderEngine(blocks=blocks, embedding=emb, final_gamma=torch.ones(BERT["hidden"], device="cuda"),
                          final_beta=torch.zeros(BERT["hidden"], device="cuda"), batch=BERT["batch"],
                          seq=BERT["seq"], causal=False,
                          lanes=lanes if lanes is not None else int(os.environ.get("ZQ_LANES", "1")))
    return eng


def gemm_roofline(torch, eng, peaks, basis):
    """Per-launch time of the fused W8A8 linears of one forward: the calls are
    recorded from an eager forward, replayed back to back in a CUDA graph (the
    same buffers, so the same work) and timed with CUDA events on the replay
    stream — no host launch gaps or per-call event overhead in the figure.  Each
    launch is bounded by max(ops / P_int8, bytes / B_hbm); at
    BERT-base shapes the f32 outputs make three of the four GEMMs HBM-bound, so
    the line reports algorithmic bytes / launch time against the HBM peak, with
    the tensor-side rate and the per-launch roofline fraction alongside."""
    calls = []
    engines = eng._sub or [eng]
    origs = [e._linear for e in engines]

    def make_rec(orig):
        def rec(q, s, w, bias, out):
            orig(q, s, w, bias, out)
            calls.append((orig, (q, s, w, bias, out)))
        return rec

    origs_ln = [e._linear_ln for e in engines]

    def make_rec_ln(orig):
        def rec(*a):
            ok = orig(*a)
            if ok:
                calls.append((orig, a))
            return ok
        return rec

    for e, o, ol in zip(engines, origs, origs_ln):
        e._linear = make_rec(o)
        e._linear_ln = make_rec_ln(ol)
    try:
        for e in engines:
            e._run()
        torch.cuda.synchronize()
    finally:
        for e, o, ol in zip(engines, origs, origs_ln):
            e._linear = o
            e._linear_ln = ol
    ops_l, bytes_l, fab_l = [], [], []
    for f, a in calls:
        q, w = a[0], a[2]
        m, k = q.shape
        n = w.rows
        if len(a) == 5:
            out = a[4]
            nb = m * k + n * k * w.bits // 8 + m * n * out.element_size() + 4 * m + 8 * n
            wr = m * n * out.element_size()
        else:  # GEMM + residual read + LN out f32 + int8 + scales
            nb = m * k + n * k + 4 * m * n + 4 * m * n + m * n + 8 * m + 16 * n
            wr = 5 * m * n
        ops_l.append(2 * m * k * n)
        bytes_l.append(nb)
        fab_l.append(fabric_time(m, n, k, wr, 2 * m * k * n, int8_peak(peaks)))
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for f, a in calls:
            f(*a)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for f, a in calls:
                f(*a)
        g.replay()
        st.synchronize()
        reps = 10
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(st)
        for _ in range(reps):
            g.replay()
        t1.record(st)
        t1.synchronize()
    t_per_pass = t0.elapsed_time(t1) * 1e-3 / reps
    n_l = max(1, len(calls))
    ops, nbytes = sum(ops_l), sum(bytes_l)
    p_int8 = int8_peak(peaks)
    p_hbm = peaks["hbm_gbs"] * 1e9
    t_roof = sum(max(o / p_int8, nb / p_hbm) for o, nb in zip(ops_l, bytes_l))
    traffic, traffic_src = measured_traffic("bert_gemm")
    achieved = nbytes / t_per_pass / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": traffic, "traffic_source": traffic_src,
            "kernel": "zq_gemm2_kernel (W8A8 linear, tcgen05 kind::i8 CTA pairs, dequant epilogue fused)",
            "launches_per_step": n_l, "per_launch_us": 1e6 * t_per_pass / n_l,
            "timing": "one forward's linears replayed back to back in a CUDA graph, CUDA events on the replay stream",
            "algorithmic_bytes_per_launch": nbytes / n_l,
            "bound_basis": "per launch max(ops / P_int8, bytes / B_hbm): the f32 outputs make O and h4h "
                           "HBM-bound and 4hh tensor-bound at BERT-base shapes (the QKV projection runs inside "
                           "the fused QKV + attention kernel, row_kernels.qkv_attention); bytes dominate the sum",
            "tensor_tops": ops / t_per_pass / 1e12, "tensor_peak": p_int8 / 1e12,
            "frac_of_per_launch_roofline": t_roof / t_per_pass,
            "fabric_roofline": {
                "frac": sum(fab_l) / t_per_pass, "bound_us_per_launch": 1e6 * sum(fab_l) / n_l,
                "basis": FABRIC_BASIS},
            "peak_basis": f"{basis} HBM copy bandwidth; " + INT8_PEAK_BASIS.format(basis=basis, **peaks)}


# SM <-> L2 fabric of this B200, measured with tools/micro (profiles/r02/tma_read_bw.txt,
# store_bw.txt): TMA reads alone 21 TB/s; SM -> L2 writes cap at 6.4 TB/s (all SMs);
# with writes at that cap, reads get 9.7 TB/s, i.e. a written byte costs the shared
# fabric as much as 21 / 11.9 read bytes.
FABRIC_READ, FABRIC_WRITE_CAP, FABRIC_WRITE_COST = 21.0e12, 6.4e12, 11.9e12
FABRIC_BASIS = ("per launch max(ops / P_int8, writes / 6.4 TB/s, operand reads / 21 TB/s + writes / 11.9 TB/s); "
                "operand reads = A once per n-tile + B once per 256-row tile (the CTA-pair kernel's L2 -> SM "
                "traffic), writes = the f32 outputs; fabric rates measured by tools/micro/tma_read_bw.cu and "
                "store_bw.cu (profiles/r02/)")


def fabric_time(m: int, n: int, k: int, wbytes: int, ops: int, p_int8: float, bn: int | None = None) -> float:
    """Lower bound of one fused linear on the measured SM <-> L2 fabric (FABRIC_BASIS)."""
    bn = bn or (256 if n % 256 == 0 or n > 2048 else 192)
    reads = m * k * math.ceil(n / bn) + n * k * math.ceil(m / 256)
    return max(ops / p_int8, wbytes / FABRIC_WRITE_CAP, reads / FABRIC_READ + wbytes / FABRIC_WRITE_COST)


def row_kernel_costs(torch, eng, peaks):
    """In-graph cost of the fused quantize kernels of the BERT forward (north-star
    target: >= 80% of HBM): the forward graph is re-captured with one kernel
    family not launched, and the replay-time difference (L2 flushed before every
    replay, outside the events) is that family's cost inside the graph, PDL
    overlaps included — unlike ncu's serialised, cold-cache launch times.  Per
    launch: algorithmic bytes / cost against the HBM copy peak."""
    t, d, f = eng.tokens, BERT["hidden"], BERT["ffn"]
    fams = {  # engine method, launches per forward, algorithmic bytes per launch
        "gelu_quant": ("_gelu_quant", BERT["layers"], 4 * t * f + t * f + 4 * t),
        "ln_quant": ("_ln_quant", 2 * BERT["layers"] + 1, 4 * t * d * 3 + t * d + 8 * d + 4 * t),
        "tok_quant": ("_tok_quant", BERT["layers"] + 1, 4 * t * d + t * d + 4 * t),
    }
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def time_graph(reps=15):
        g = eng.capture()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        return ts[len(ts) // 2] * 1e-3

    base = time_graph()
    out = {"method": "in-graph cost = forward replay time minus the replay time with the family not launched "
                     "(median of 15, L2 flushed before each replay); bytes = algorithmic (inputs read + "
                     "outputs written once)", "forward_s": base}
    noop = lambda *a, **k: None  # noqa: E731
    for name, (attr, nl, nbytes) in fams.items():
        orig = getattr(eng, attr)
        setattr(eng, attr, noop)
        try:
            t_without = time_graph()
        finally:
            setattr(eng, attr, orig)
        per = max(base - t_without, 1e-9) / nl
        out[name] = {"launches_per_forward": nl, "in_graph_us_per_launch": 1e6 * per,
                     "algorithmic_bytes_per_launch": nbytes, "achieved_GBps": nbytes / per / 1e9,
                     "frac_of_hbm": nbytes / per / 1e9 / peaks["hbm_gbs"]}
    if eng._fuse_qkv:
        # fused QKV projection + attention (zq_qkv_attention): bounded by its tensor
        # work (int8 GEMM at P_int8 plus the 3-term f16 S and P V products at the
        # bf16 peak) since its bytes (x int8, W_qkv int8, ctx f32) are few
        orig = eng._qkv_attention
        eng._qkv_attention = lambda *a, **k: True
        try:
            t_without = time_graph()
        finally:
            eng._qkv_attention = orig
        nl = BERT["layers"]
        per = max(base - t_without, 1e-9) / nl
        units = BERT["batch"] * BERT["heads"]
        i8_ops = 2 * t * d * 3 * d
        f16_flops = units * 2 * 3 * 2 * 128 * 128 * (d // BERT["heads"])
        nbytes = t * d + 3 * d * d + 4 * 6 * d + 4 * t + 4 * t * d
        t_bound = max(i8_ops / int8_peak(peaks) + f16_flops / (peaks["bf16_tflops"] * 1e12),
                      nbytes / (peaks["hbm_gbs"] * 1e9))
        out["qkv_attention"] = {
            "kernel": "qkv_attention_kernel (W8A8 QKV GEMM tcgen05 kind::i8 + fp16 two-term attention, one "
                      "(sequence, head) unit per CTA step; the f32 QKV never reaches HBM)",
            "launches_per_forward": nl, "in_graph_us_per_launch": 1e6 * per,
            "int8_ops_per_launch": i8_ops, "f16_flops_per_launch": f16_flops,
            "algorithmic_bytes_per_launch": nbytes, "bound_us": 1e6 * t_bound, "frac_of_roofline": t_bound / per,
            "bound_basis": "int8 ops / P_int8 + f16 flops / bf16 peak (tensor-bound; bytes / B_hbm is smaller)"}
    eng.capture()  # leave the engine with its full graph
    del flush
    return out


INT8_NOMINAL_TOPS = 4500.0
INT8_PEAK_BASIS = ("P_int8 = 2 x {basis} cuBLAS bf16 dense ({bf16_tflops} TF/s): tcgen05 kind::i8 issues at twice "
                   "the kind::f16 rate, so this is the int8 rate a cuBLAS-grade kernel reaches here; the nominal "
                   "dense INT8 peak is 4500 TOPS (frac_of_nominal)")


def int8_peak(peaks) -> float:
    """ops/s denominator for the int8 tensor roofline (see INT8_PEAK_BASIS)."""
    return 2.0 * peaks["bf16_tflops"] * 1e12


def measured_traffic(key: str):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of the
    named kernel family from the ncu --set full capture recorded in
    profiles/traffic.json (averaged over the family's launches in one forward),
    with its provenance; (None, reason) when no capture is recorded."""
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(tp):
        return None, "no ncu capture recorded"
    with open(tp) as f:
        d = json.load(f)
    e = d.get(key)
    if not isinstance(e, dict):
        return None, "no ncu capture recorded for " + key
    return e["bytes_per_launch"], e["source"]


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
    torch.cuda.nvtx.range_push("bench_timed")  # ncu --nvtx-include "bench_timed/" selects these launches
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            eng.launch()
            b.record(stream)
            times.append((a, b))
        barrier()
    torch.cuda.nvtx.range_pop()
    step_s = [a.elapsed_time(b) * 1e-3 for a, b in times]
    total = sum(step_s)
    eng.check_finite()

    # ---- end to end through the public API with host buffers ----
    # Every step: an H2D of the step's token ids from pinned host memory, the
    # forward (EncoderEngine.forward), and a D2H of the step's hidden states.  As
    # in a serving pipeline, step i+1's ids travel on an upload stream while step
    # i computes (forward() then takes them device to device), and the D2H of step
    # i runs on a copy stream while step i+1 computes: two engines over the same
    # weights take alternate steps (double-buffered outputs, as a server would
    # run), so step i's hidden states are read straight from its engine's output
    # buffer while the other engine computes.  The D2H is issued once step i+1's
    # L2 flush has finished, so it overlaps the forward rather than the flush
    # (whose own time is subtracted); the timed region spans all steps, from the
    # first upload to the last D2H.
    from paper_2206_01861_b200 import transformer as T

    eng2 = T.EncoderEngine(blocks=eng.blocks, embedding=eng.embedding, final_gamma=eng.final_gamma,
                           final_beta=eng.final_beta, batch=eng.batch, seq=eng.seq, causal=eng.causal,
                           lanes=eng.lanes)
    engs = [eng, eng2]
    for e_ in engs:  # capture both graphs outside the timed region
        e_.forward(ids_host)
    torch.cuda.synchronize()
    out_host = [torch.empty((eng.tokens, BERT["hidden"]), dtype=torch.float32).pin_memory() for _ in range(2)]
    outs = [None, None]
    copy_stream = torch.cuda.Stream()
    up_stream = torch.cuda.Stream()
    ids_dev = [torch.empty_like(ids_host, device="cuda") for _ in range(2)]
    uploaded = [None, None]
    consumed = [None, None]
    copied = [None, None]
    pending = None  # (slot, ready event) of the step whose D2H is still to be issued

    def upload(slot):
        if consumed[slot] is not None:
            up_stream.wait_event(consumed[slot])  # the forward that read this slot has copied it
        with torch.cuda.stream(up_stream):
            ids_dev[slot].copy_(ids_host, non_blocking=True)  # H2D of a step's ids
        uploaded[slot] = torch.cuda.Event()
        uploaded[slot].record(up_stream)

    def issue_d2h(slot, ready):
        copy_stream.wait_event(ready)
        with torch.cuda.stream(copy_stream):
            out_host[slot].copy_(outs[slot], non_blocking=True)  # D2H of the result
        copied[slot] = torch.cuda.Event()
        copied[slot].record(copy_stream)

    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush_ev = []
    a.record(stream)
    up_stream.wait_event(a)
    upload(0)
    for i in range(args.steps):
        fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fa.record(stream)
        flush.zero_()                        # timed separately and subtracted below
        fb.record(stream)
        flush_ev.append((fa, fb))
        if pending is not None:              # previous step's D2H, after this flush
            copy_stream.wait_event(fb)
            issue_d2h(*pending)
        j = i % 2
        stream.wait_event(uploaded[j])
        if copied[j] is not None:
            stream.wait_event(copied[j])     # the D2H that read this engine's output is done
        outs[j] = engs[j].forward(ids_dev[j])  # ids device to device, then the forward graph
        consumed[j] = torch.cuda.Event()
        consumed[j].record(stream)
        if i + 1 < args.steps:
            upload((i + 1) % 2)              # the next step's ids, during this forward
        ready = torch.cuda.Event()
        ready.record(stream)
        pending = (j, ready)
    issue_d2h(*pending)
    stream.wait_stream(copy_stream)
    b.record(stream)
    barrier()
    flush_total = sum(x.elapsed_time(y) for x, y in flush_ev) * 1e-3
    e2e_total = a.elapsed_time(b) * 1e-3 - flush_total

    if dist is not None:
        t = torch.tensor([total, e2e_total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total, e2e_total = float(t[0]), float(t[1])

    seqs = BERT["batch"] * world * args.steps
    value = seqs / total
    e2e_value = seqs / e2e_total
    roof = gemm_roofline(torch, eng, peaks, basis) if rank == 0 else None
    rows = row_kernel_costs(torch, eng, peaks) if rank == 0 and not eng._sub else None
    fused = all(e._fuse_ln for e in (eng._sub or [eng]))
    fused_qkv = all(e._fuse_qkv for e in (eng._sub or [eng]))
    clocks = clk.summary()
    step_mm = [1000 * min(step_s), 1000 * max(step_s)]
    ids_bytes, out_bytes = int(ids_host.numel() * 8), int(out_host[0].numel() * 4)
    del eng, eng2, engs, outs, out_host, flush
    torch.cuda.empty_cache()
    extra = secondary_workloads(rank, world, dist) if args.workload == "all" else None
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    cpu_val, cpu_sample, _ = cpu_reference_sample(cores, 1)
    # tok quant + per block (QKV GEMM + attention fused: one launch fewer; linear + LN fused: two fewer) + final LN
    launches_per_step = 2 + (9 - (1 if fused_qkv else 0) - (2 if fused else 0)) * BERT["layers"]
    line = {
        "metric": "BERT-base W8A8 encoder forward throughput", "value": value, "unit": "seq/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int8", "data": "synthetic (random-init weights, random token ids)",
        "config": workload_config(),
        "e2e": {"value": e2e_value, "unit": "seq/s", "h2d_bytes_per_step": ids_bytes,
                "d2h_bytes_per_step": out_bytes,
                "pipeline": "two engines over the same weights take alternate steps (double-buffered outputs); step i+1's token ids upload on their own stream during step i, and the D2H of step i's hidden states (straight from its engine's output) overlaps step i+1 on a copy stream; an L2 flush (256 MiB memset) precedes every step, its own event-timed duration subtracted"},
        "roofline": roof,
        "row_kernels": rows,
        "cpu_baseline": {"value": cpu_val, "unit": "seq/s", "cores": cores, "kind": "port", "sample": cpu_sample},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "step_ms_min_max": step_mm,
    }
    if extra is not None:
        line["workloads"] = extra
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPT workloads (BASELINE configs 2-4): prefill + greedy decode with KV cache
# ---------------------------------------------------------------------------

GPT_RUNS = {
    # name: (batch, prompt tokens, new tokens)
    "gpt3-350m": (8, 1024, 16),
    "gptj-6b": (16, 128, 128),
    "neox-20b": (16, 128, 128),
}


def _gpt_ref_worker(args):
    """Reference algorithm (oracle port) on one sequence of `t` tokens through one
    block of the named GPT shape: returns seconds."""
    name, t, seed = args
    import numpy as np

    from oracle import lowbit_oracle as O
    from paper_2206_01861_b200.decoder import CONFIGS

    cfg = CONFIGS[name]
    O.use_reference_cost_igemm(True)
    d, f = cfg.dim, cfg.ffn
    rng = np.random.default_rng(seed)  # fast generator: only the block's cost is measured
    w = {n: (rng.standard_normal(s, dtype=np.float32) * np.float32(0.02)) for n, s in (
        ("w_q", (d, d)), ("w_k", (d, d)), ("w_v", (d, d)), ("w_o", (d, d)),
        ("w_h4h", (f, d)), ("w_4hh", (d, f)))}
    for n, s in (("b_q", d), ("b_k", d), ("b_v", d), ("b_o", d), ("b_h4h", f), ("b_4hh", d),
                 ("ln1_beta", d), ("ln2_beta", d)):
        w[n] = np.zeros(s, np.float32)
    w["ln1_gamma"] = np.ones(d, np.float32)
    w["ln2_gamma"] = np.ones(d, np.float32)
    qb = O.quantize_block(w, cfg.mhsa_bits, cfg.ffc_bits, cfg.groups)
    x = O.Rng(seed + 1).gaussian((t, d), std=0.5)
    t0 = time.perf_counter()
    O.block_forward(x, qb, cfg.heads, True, "int8")
    return time.perf_counter() - t0


def gpt_cpu_sample(name: str, cores: int):
    """Reference CPU throughput estimate for the generation workload: the
    reference recomputes the full context per generated token (evaluate.py:96-98),
    so a generated token costs one causal forward over the context.  Sample: one
    block over a 16-token sequence per core (bounded), scaled linearly in tokens
    (the int64 igemm dominates and is linear in tokens) and x layers."""
    from concurrent.futures import ProcessPoolExecutor

    from paper_2206_01861_b200.decoder import CONFIGS

    cfg = CONFIGS[name]
    batch, prompt, new = GPT_RUNS[name]
    ts = 8
    with ProcessPoolExecutor(max_workers=1) as ex:  # one core: a GPT-scale block is ~GBs of host RAM
        secs = list(ex.map(_gpt_ref_worker, [(name, ts, 1)]))
    cores = 1
    per_tok_layer = statistics.median(secs) / ts
    # tokens processed by recomputation: sum over steps of the context length
    ctx_tokens = batch * sum(prompt + i for i in range(new))
    total_s = per_tok_layer * cfg.layers * ctx_tokens / cores
    value = batch * new / total_s
    sample = (f"1 process x 1 {cfg.name} block over {ts} tokens (reference numpy algorithm, int64 "
              f"igemm); x{cfg.layers} layers, x full-context recomputation per generated token "
              f"(evaluate.py:96-98), extrapolated")
    return value, sample, cores


def gpt_measure(name: str, steps: int, warmup: int, rank: int, world: int, dist, cpu: bool = True):
    """One GPT generation workload (BASELINE configs[2-4]): batch x prompt
    prefill + (new - 1) KV-cached greedy decode steps per step, tensor parallel
    over all `world` ranks (Megatron; tp.row_parallel_linear).  Returns rank 0's
    line (None on the other ranks)."""
    import numpy as np
    import torch

    from paper_2206_01861_b200.decoder import CONFIGS, DecoderEngine

    cfg = CONFIGS[name]
    batch, prompt, new = GPT_RUNS[name]
    tp = (None, rank, world) if world > 1 else None
    eng = DecoderEngine(cfg, batch, prompt + new, seed=0, tp=tp)
    ids_host = torch.from_numpy(np.random.default_rng(0).integers(0, cfg.vocab, (batch, prompt))).pin_memory()
    ids_dev = ids_host.cuda()
    out_host = torch.empty((batch, new), dtype=torch.int64).pin_memory()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def generate(ids):
        toks = [eng.prefill(ids).clone()]
        for _ in range(new - 1):
            toks.append(eng.step().clone())
        return torch.stack(toks, 1)

    for _ in range(warmup):
        generate(ids_dev)
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    pre_t, dec_t = [], []
    barrier()
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(steps):
            flush.zero_()
            a, m, b = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record(stream)
            toks = [eng.prefill(ids_dev).clone()]
            m.record(stream)
            for _ in range(new - 1):
                toks.append(eng.step().clone())
            b.record(stream)
            pre_t.append((a, m))
            dec_t.append((m, b))
        barrier()
    prefill_s = sum(x.elapsed_time(y) for x, y in pre_t) * 1e-3
    decode_s = sum(x.elapsed_time(y) for x, y in dec_t) * 1e-3
    total = prefill_s + decode_s
    eng.check_finite()
    # end to end: pinned host ids -> tokens back in pinned host memory, every step
    barrier()
    e2e = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out_host.copy_(generate(ids_host), non_blocking=True)
        b.record(stream)
        e2e.append((a, b))
    barrier()
    e2e_s = sum(x.elapsed_time(y) for x, y in e2e) * 1e-3
    # our kernel launches per generation: count the C-ABI entry points one eager
    # prefill and one eager decode step make (each launches one kernel; the
    # embedding gather is a torch op, not ours).  transformer.attention wraps
    # zq_attention_f32 and is counted there.
    from paper_2206_01861_b200 import _native as N
    from paper_2206_01861_b200 import decoder as D
    calls = {"n": 0}
    orig_call, orig_att, orig_rc = N.call, D.attention, N.call_rc

    def counting_call(nm, *a):
        calls["n"] += 1
        return orig_call(nm, *a)

    def counting_att(*a, **kw):
        calls["n"] += 1
        return orig_att(*a, **kw)

    def counting_rc(nm, *a):
        rc = orig_rc(nm, *a)
        if rc == 0:
            calls["n"] += 1
        return rc

    N.call, N.call_rc, D.attention = counting_call, counting_rc, counting_att
    try:
        eng.prefill(ids_dev)
        n_prefill = calls["n"]
        calls["n"] = 0
        eng._step_launches()
        n_step = calls["n"]
    finally:
        N.call, N.call_rc, D.attention = orig_call, orig_rc, orig_att
    torch.cuda.synchronize()
    launches = steps * (n_prefill + (new - 1) * n_step)
    if dist is not None:
        t = torch.tensor([total, prefill_s, decode_s, e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total, prefill_s, decode_s, e2e_s = (float(v) for v in t)
    # roofline of the decode step: what one rank must stream from HBM per token
    # step — its int8 (or packed int4) weights, plus the f32 K/V cache rows the
    # decode attention reads (the average context over the decode steps)
    wbytes = 0
    for blk in eng.blocks:
        for wn in ("w_qkv", "w_o", "w_h4h", "w_4hh"):
            w = getattr(blk, wn)
            wbytes += w.rows * w.ld * (w.bits / 8)
    avg_ctx = prompt + new / 2.0
    kvbytes = len(eng.blocks) * 2 * batch * avg_ctx * eng.dl * 4
    emb_bytes = cfg.vocab * cfg.dim * 4  # tied LM head (f32 embedding), every step
    step_bytes = wbytes + kvbytes + emb_bytes
    del eng
    torch.cuda.empty_cache()
    if rank != 0:
        return None
    peaks, basis = load_peaks()
    step_s = decode_s / (steps * (new - 1))
    achieved = step_bytes / step_s / 1e9
    toks = batch * new * steps
    line = {
        "metric": f"{cfg.name} greedy generation throughput", "value": toks / total, "unit": "tok/s",
        "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": 1000 * total / steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int8",
        "data": "synthetic (random-init weights, random prompt ids)",
        "config": {"workload": f"{cfg.name}: batch {batch}, prompt {prompt}, {new} new tokens (greedy, KV cache)",
                   "layers": cfg.layers, "hidden": cfg.dim, "heads": cfg.heads, "ffn": cfg.ffn,
                   "weight_bits": [cfg.mhsa_bits, cfg.ffc_bits], "weight_groups": cfg.groups,
                   "parallelism": f"tp{world}" if world > 1 else "single",
                   "l2": "flushed (256 MiB memset) before each generation"},
        "prefill_tok_per_s": batch * prompt * steps / prefill_s,
        "decode_ms_per_token": 1000 * step_s,
        "e2e": {"value": toks / e2e_s, "unit": "tok/s", "h2d_bytes_per_step": int(ids_host.numel() * 8),
                "d2h_bytes_per_step": int(out_host.numel() * 8)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                     "kernel": "decode step (per rank): int8 weight streaming of the quantized linears + f32 KV "
                               "cache reads of decode attention + f32 tied LM head",
                     "bytes_per_step": step_bytes, "weight_bytes": wbytes, "kv_bytes": kvbytes,
                     "lm_head_bytes": emb_bytes, "kv_basis": f"average context {avg_ctx:.0f} tokens",
                     "peak_basis": f"{basis} HBM copy bandwidth (MEASURED_PEAKS.json)"},
        "gpu_launches": launches,
        "gpu_launches_per": {"prefill": n_prefill, "decode_step": n_step},
        "clocks": clk.summary(),
    }
    if cpu:
        cpu_val, cpu_sample, cores = gpt_cpu_sample(name, len(os.sched_getaffinity(0)))
        line["cpu_baseline"] = {"value": cpu_val, "unit": "tok/s", "cores": cores, "kind": "port",
                                "sample": cpu_sample}
    return line


def c1_measure(steps: int, warmup: int, rank: int, world: int, out_dtype=None):
    """BASELINE configs[0]: one W8A8 quantized linear 768->3072 over 32x128 tokens
    (fp32 in; f32 out, or fp16 with out_dtype=torch.float16), activation
    quantization included; metric = TOPS.  Replicas across ranks."""
    import torch

    from paper_2206_01861_b200 import _native as N
    from paper_2206_01861_b200 import igemm, quant

    out_dtype = out_dtype or torch.float32
    t, k, n, g = 4096, 768, 3072, 48
    gen = torch.Generator(device="cuda").manual_seed(rank)
    sets = [torch.randn((t, k), generator=gen, device="cuda") for _ in range(8)]  # 8 x 12.6 MB rotating
    w = quant.quantize_weight_groupwise(torch.randn((n, k), generator=gen, device="cuda") * 0.02, g, 8)
    bias = torch.zeros(n, device="cuda")
    out = torch.empty((t, n), device="cuda", dtype=out_dtype)
    q = quant.padded_int8(t, k)
    s = torch.empty(t, device="cuda")
    fl = quant.FiniteFlag()
    wp, ldw, wb = w.weight_operand()
    code = igemm._OUT_CODES[out_dtype]

    def step(x):
        N.call("zq_quantize_tokenwise", x.data_ptr(), t, k, k, 8, q.data_ptr(), q.stride(0), s.data_ptr(),
               fl.ptr, N.stream_ptr())
        N.call("zq_linear", q.data_ptr(), q.stride(0), s.data_ptr(), 0.0, wp, ldw, wb, w.row_scales().data_ptr(),
               bias.data_ptr(), t, n, k, out.data_ptr(), out.stride(0), code, N.stream_ptr())

    for i in range(warmup):
        step(sets[i % 8])
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    # the K timed steps (rotating over 8 inputs, 100 MB > what one step touches)
    # captured back to back in one CUDA graph: no host launch gaps between steps
    g_ = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_):
        for i in range(steps):
            step(sets[i % 8])
    g_.replay()  # warm
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g_.replay()
        b.record(stream)
        torch.cuda.synchronize()
    sec = a.elapsed_time(b) * 1e-3 / steps
    ops = 2 * t * k * n
    ob = out.element_size()
    c1_bytes = t * k * 4 + 2 * (t * k + 4 * t) + n * k + 8 * n + t * n * ob
    x_host = torch.randn((t, k)).pin_memory()
    o_host = torch.empty((t, n), dtype=out_dtype).pin_memory()
    for _ in range(max(warmup, 3)):  # untimed: first-use costs of the eager path and the pinned buffers
        o_host.copy_(igemm.quantized_linear(x_host.cuda(non_blocking=True), w, bias, igemm.DynamicAct(8),
                                            out_dtype=out_dtype), non_blocking=True)
    torch.cuda.synchronize()
    ev = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        xd = x_host.cuda(non_blocking=True)
        o_host.copy_(igemm.quantized_linear(xd, w, bias, igemm.DynamicAct(8), out_dtype=out_dtype), non_blocking=True)
        b.record(stream)
        ev.append((a, b))
    torch.cuda.synchronize()
    e2e = sum(a.elapsed_time(b) for a, b in ev) * 1e-3 / steps
    if rank != 0:
        return None
    peaks, basis = load_peaks()
    p8 = int8_peak(peaks)
    dt = {torch.float32: "f32", torch.float16: "f16", torch.bfloat16: "bf16"}[out_dtype]
    return {"metric": f"ZeroQuant W8A8 quantized linear throughput ({dt} out, incl. token-wise activation quantization)",
            "value": world * ops / sec / 1e12, "unit": "TOPS", "n_gpus": world, "steps": steps,
            "warmup": warmup, "ms_per_step": 1000 * sec, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int8", "data": "synthetic",
            "config": {"workload": f"BASELINE configs[0]: 4096 tokens x 768 -> 3072, groups 48, f32 in, {dt} out",
                       "l2": "8 rotating 12.6 MB inputs; K steps replayed as one CUDA graph"},
            "e2e": {"value": world * ops / e2e / 1e12, "unit": "TOPS", "h2d_bytes_per_step": t * k * 4,
                    "d2h_bytes_per_step": t * n * ob},
            # step = token quantize (x f32 in, int8 + scales out) + fused linear (int8 in, out):
            # max(ops / P_int8, bytes / B_hbm) says HBM for f32 out
            "roofline": {"bound": "hbm" if c1_bytes / (1e9 * peaks["hbm_gbs"]) > ops / p8 else "tensor",
                         "achieved": c1_bytes / sec / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": c1_bytes / sec / 1e9 / peaks["hbm_gbs"], "traffic": None,
                         "algorithmic_bytes_per_step": c1_bytes,
                         "tensor_tops": ops / sec / 1e12, "tensor_peak": p8 / 1e12,
                         "frac_of_int8_nominal": ops / sec / 1e12 / INT8_NOMINAL_TOPS,
                         "frac_of_roofline": max(ops / p8, c1_bytes / (1e9 * peaks["hbm_gbs"])) / sec,
                         "peak_basis": f"{basis} HBM copy bandwidth; " + INT8_PEAK_BASIS.format(basis=basis, **peaks)},
            "gpu_launches": 2 * steps, "clocks": clk.summary()}


GEMM_LARGE = [  # (label, M tokens, N out, K in)
    ("8192^3", 8192, 8192, 8192),
    ("NeoX-20B prefill h4h (16x128 tokens)", 2048, 24576, 6144),
    ("NeoX-20B prefill 4hh (16x128 tokens)", 2048, 6144, 24576),
    ("GPT-J 6B prefill h4h (16x128 tokens)", 2048, 16384, 4096),
]


def gemm_large_measure(steps: int, warmup: int, rank: int, world: int):
    """North-star target check: the fused W8A8 quantized linear (int8 activations
    with token scales -> tcgen05 kind::i8 -> exact dequant epilogue, f32 out) at
    large shapes, in TOPS against the INT8 peak.  Per shape: `steps` launches
    captured in one CUDA graph, timed with CUDA events; 2 operand sets rotate so
    consecutive launches do not reuse an L2-resident operand."""
    import torch

    from paper_2206_01861_b200 import _native as N
    from paper_2206_01861_b200 import quant

    peaks, basis = load_peaks()
    p8 = int8_peak(peaks)
    res = []
    gen = torch.Generator(device="cuda").manual_seed(7 + rank)
    for label, m, n, k in GEMM_LARGE:
        sets = []
        for _ in range(2):
            xq = quant.padded_int8(m, k)
            xq.copy_(torch.randint(-127, 128, (m, k), generator=gen, device="cuda", dtype=torch.int8))
            ws = quant.padded_int8(n, k, align=32)
            ws.copy_(torch.randint(-127, 128, (n, k), generator=gen, device="cuda", dtype=torch.int8))
            sets.append((xq, ws, torch.rand(m, device="cuda") * 0.01 + 1e-3))
        rs = torch.rand(n, device="cuda") * 1e-3 + 1e-4
        bias = torch.zeros(n, device="cuda")
        out = torch.empty((m, n), device="cuda")

        def launch(i):
            xq, ws, ts = sets[i % 2]
            N.call("zq_linear", xq.data_ptr(), xq.stride(0), ts.data_ptr(), 0.0, ws.data_ptr(), ws.stride(0), 8,
                   rs.data_ptr(), bias.data_ptr(), m, n, k, out.data_ptr(), out.stride(0), N.OUT_F32, N.stream_ptr())

        for i in range(warmup):
            launch(i)
        torch.cuda.synchronize()
        g_ = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_):
            for i in range(steps):
                launch(i)
        g_.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(torch.cuda.current_device()) as clk:
            a.record()
            g_.replay()
            b.record()
            torch.cuda.synchronize()
        sec = a.elapsed_time(b) * 1e-3 / steps
        ops = 2 * m * n * k
        nbytes = m * k + n * k + 4 * m * n + 4 * m + 8 * n
        res.append({"shape": label, "M": m, "N": n, "K": k, "us": 1e6 * sec, "tops": ops / sec / 1e12,
                    "frac_of_int8_peak": ops / sec / p8, "frac_of_int8_nominal": ops / sec / 1e12 / INT8_NOMINAL_TOPS,
                    "bound": "tensor" if ops / p8 > nbytes / (1e9 * peaks["hbm_gbs"]) else "hbm",
                    "clocks": clk.summary()})
        del sets, out
        torch.cuda.empty_cache()
    if rank != 0:
        return None
    best = max(res, key=lambda r: r["tops"])
    return {"metric": "W8A8 quantized linear TOPS at large shapes (vs INT8 peak)", "value": world * best["tops"],
            "unit": "TOPS", "n_gpus": world, "steps": steps, "warmup": warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic int8 operands",
            "config": {"workload": "fused W8A8 linear (tcgen05 kind::i8, exact dequant epilogue, f32 out); "
                                   "value = best shape, per shape below"},
            "shapes": res,
            "roofline": {"bound": "tensor", "achieved": best["tops"], "peak": p8 / 1e12, "unit": "TFLOP/s",
                         "frac": best["frac_of_int8_peak"], "traffic": None,
                         "peak_basis": INT8_PEAK_BASIS.format(basis=basis, **peaks)}}


WO_SHAPES = [("NeoX-20B QKV prefill", 2048, 18432, 6144), ("NeoX-20B h4h prefill", 2048, 24576, 6144),
             ("NeoX-20B 4hh prefill", 2048, 6144, 24576)]


def wo_gemm_measure(steps: int, warmup: int, rank: int, world: int):
    """The tensor-core FullAct (weight-only, W8A16 / the A16 sites of W8A8/16)
    linear at NeoX-20B prefill shapes (batch 16 x 128 tokens): activation split
    (f32 -> power-of-two-scaled f16 terms) + the converted-weight CTA-pair GEMM
    (int8 weights -> f16 in smem, tcgen05 kind::f16), f16 out.  TFLOP/s against
    the measured bf16 dense peak; `steps` launches per shape in one CUDA graph."""
    import torch

    from paper_2206_01861_b200 import _native as N
    from paper_2206_01861_b200 import quant

    peaks, basis = load_peaks()
    pbf = peaks["bf16_tflops"] * 1e12
    res = []
    gen = torch.Generator(device="cuda").manual_seed(11 + rank)
    for label, m, n, k in WO_SHAPES:
        for wbits, terms in ((8, 1), (8, 2), (4, 1)):
            w = torch.randn(n, k, generator=gen, device="cuda") * 0.02
            wq = quant.quantize_weight_groupwise(w, 128, wbits)
            del w
            xs = [torch.randn(m, k, generator=gen, device="cuda") for _ in range(2)]
            ld_h = (k + 7) // 8 * 8
            hi = torch.empty(m, ld_h, dtype=torch.float16, device="cuda")
            lo = torch.empty(m, ld_h, dtype=torch.float16, device="cuda") if terms == 2 else None
            ri = torch.empty(m, device="cuda")
            out = torch.empty(m, n, dtype=torch.float16, device="cuda")
            wp, ld_w, wb = wq.weight_operand()
            rs = wq.row_scales()

            def launch(i):
                x = xs[i % 2]
                N.call("zq_act_split16", x.data_ptr(), x.stride(0), m, k, terms, hi.data_ptr(), N.ptr(lo), ld_h,
                       ri.data_ptr(), None, N.stream_ptr())
                N.call("zq_linear_wo", hi.data_ptr(), N.ptr(lo), ld_h, ri.data_ptr(), wp, ld_w, wb, rs.data_ptr(),
                       None, m, n, k, out.data_ptr(), out.stride(0), N.OUT_F16, N.stream_ptr())

            for i in range(warmup):
                launch(i)
            torch.cuda.synchronize()
            g_ = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_):
                for i in range(steps):
                    launch(i)
            g_.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with ClockSampler(torch.cuda.current_device()) as clk:
                a.record()
                g_.replay()
                b.record()
                torch.cuda.synchronize()
            sec = a.elapsed_time(b) * 1e-3 / steps
            fl = 2.0 * m * n * k
            res.append({"shape": label, "M": m, "N": n, "K": k, "w_bits": wbits,
                        "mode": "f16" if terms == 1 else "f16x2", "us": 1e6 * sec, "tflops": fl / sec / 1e12,
                        "frac_of_bf16_peak": fl / sec / pbf, "clocks": clk.summary()})
            del xs, hi, lo, out, wq
            torch.cuda.empty_cache()
    if rank != 0:
        return None
    w8 = [r for r in res if r["w_bits"] == 8 and r["mode"] == "f16"]
    best = max(w8, key=lambda r: r["tflops"])
    return {"metric": "W8A16 weight-only linear TFLOP/s at NeoX-20B prefill shapes (vs bf16 peak)",
            "value": world * best["tflops"], "unit": "TFLOP/s", "n_gpus": world, "steps": steps, "warmup": warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic", "config": {"workload": "FullAct tensor-core mode: act split + converted-weight "
                                                        "pair GEMM, f16 out; value = best W8 f16 shape, per shape below",
                                            "l2": "2 rotating activation inputs; weights 113-302 MB (> L2)"},
            "shapes": res,
            "roofline": {"bound": "tensor", "achieved": best["tflops"], "peak": pbf / 1e12, "unit": "TFLOP/s",
                         "frac": best["frac_of_bf16_peak"], "traffic": None,
                         "peak_basis": f"measured bf16 dense ({basis})"}}


SECONDARY = ("c1", "c1-f16", "gemm-large", "wo-gemm", "gpt3-350m", "gptj-6b", "neox-20b")


def secondary_workloads(rank: int, world: int, dist):
    """The other BASELINE configurations, measured in the same run as the
    headline (bounded step counts).  A failure is recorded in place; it does
    not void the headline."""
    import torch

    out = {}
    for name in SECONDARY:
        t0 = time.time()
        try:
            if name == "c1":
                r = c1_measure(20, 5, rank, world)
            elif name == "c1-f16":
                r = c1_measure(20, 5, rank, world, out_dtype=torch.float16)
            elif name == "gemm-large":
                r = gemm_large_measure(10, 3, rank, world)
            elif name == "wo-gemm":
                r = wo_gemm_measure(10, 3, rank, world)
            else:
                r = gpt_measure(name, 2, 3, rank, world, dist, cpu=False)
        except Exception as e:  # noqa: BLE001 - recorded, the headline stands
            r = {"error": f"{type(e).__name__}: {e}"[:400]}
        torch.cuda.empty_cache()
        if r is not None:
            r["wall_s"] = round(time.time() - t0, 1)
            out[name] = r
    return out


def run_single(args, rank: int, world: int, dist):
    """--workload X (not bert/all): X's own JSON line."""
    import torch

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    if args.workload in ("c1", "c1-f16"):
        line = c1_measure(args.steps, args.warmup, rank, world,
                          out_dtype=torch.float16 if args.workload == "c1-f16" else None)
    elif args.workload == "gemm-large":
        line = gemm_large_measure(args.steps, args.warmup, rank, world)
    elif args.workload == "wo-gemm":
        line = wo_gemm_measure(args.steps, args.warmup, rank, world)
    else:
        line = gpt_measure(args.workload, args.steps, args.warmup, rank, world, dist)
    if line is not None:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="all", choices=["all", "bert"] + list(SECONDARY))
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
        import datetime

        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl", timeout=datetime.timedelta(seconds=600))
        dist = tdist
    if args.workload in ("all", "bert"):
        run_ours(args, rank, world, dist)
    else:
        run_single(args, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
