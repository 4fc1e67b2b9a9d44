#!/usr/bin/env python
"""DSA attention tokens/s (predict + select + sparse attention) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2_vector]
    python bench.py --impl reference ...      # the reference CPU path

One JSON line on rank 0.  A "step" is one pass of the hot path over the
config's full batch: all B*H (b,h) pairs, phases 1 -> 2 -> 3, inputs resident
in HBM (`value`), or through the C-ABI with host buffers and H2D/D2H copies
inside the timed region (`e2e`).  With N GPUs the config's B*H pairs are
partitioned over the ranks (strong scaling): rank r runs
shard.pair_range(r, N, B*H) with no collective on the hot path; the time is
the max over ranks; per-pair checksums are all-gathered over NCCL after
timing stops.  `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks.
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
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DSA attention tokens/s (predict+sparse attn) at L=4096, 95% sparsity; % roofline"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return d, "measured (MEASURED_PEAKS.json)"
    return dict(PEAKS_FALLBACK), "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL needs one GPU per rank; more ranks than GPUs (a 1-GPU box
        # checking the partition logic) or a CPU run fall back to gloo
        ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
        backend = os.environ.get("DSA_BENCH_BACKEND") or ("nccl" if ndev >= world else "gloo")
        dist.init_process_group(backend)
    return rank, local, world


def dist_device(device):
    """Device for collective tensors: the GPU under NCCL, the host under gloo."""
    import torch.distributed as dist
    return device if dist.get_backend() == "nccl" else "cpu"


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dist_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- CPU arms
REF_MODES = {"row_topk": 0, "colvec": 1, "block": 2, "threshold": 3}


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_inputs(p, pair0: int, npairs: int):
    """The config's seeded inputs drawn with the REFERENCE Rng (oracle/_ref,
    ref_generate; bit-identical to dsa_generate, tests/test_oracle.py) -- the
    reference arm never loads libdsa_b200.so."""
    from oracle.oracle import Reference
    return Reference().generate(p.L, p.d, p.k, p.dtype == "bf16", p.seed, p.planted_per_mille,
                                p.band_width, pair0, npairs)


def reference_run(p, inputs, threads: int) -> float:
    """One pass of the reference implementation (oracle/_ref: the unmodified
    reference sources + extern "C" compositions of reference functions) over
    the pairs in `inputs`, on `threads` host threads; returns wall seconds."""
    from oracle.oracle import Reference
    ref = Reference()
    q, k, v, P = inputs
    t0 = time.perf_counter()
    ref.pipeline(q, k, v, P, p.bits, p.dtype == "f32", REF_MODES[p.mask_mode], p.keep, p.vec_v, p.block,
                 p.force_diag, threads=threads, per_row=p.quant_scope == "row", frac_num=p.frac_num,
                 frac_den=p.frac_den, cap=p.cap, causal=p.causal)
    return time.perf_counter() - t0


def reference_pairs(p, threads: int) -> int:
    """Pairs per reference step: every pair for C0-C2 (L <= 4096, BASELINE.md
    2); a bounded sample of C3/C4 (seconds of CPU work per pair), so the whole
    --impl reference run ends within minutes."""
    if p.L <= 4096:
        return p.pairs
    return min(p.pairs, max(1, threads))


def run_reference_arm(args, p, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    npairs = min(p.pairs, args.ref_pairs) if args.ref_pairs else reference_pairs(p, threads)
    inputs = reference_inputs(p, 0, npairs)
    tokens = npairs * p.L / p.heads
    for _ in range(args.warmup):
        reference_run(p, inputs, threads)
    times = [reference_run(p, inputs, threads) for _ in range(args.steps)]
    mean = statistics.mean(times)
    value = tokens / mean
    from oracle.oracle import Reference
    isa = Reference().isa()
    sample = (f"{npairs} of {p.pairs} (b,h) pairs per step through oracle/_ref (the reference sources, "
              f"isa={isa}; inputs from the reference Rng); tokens = pairs*L/heads; cpu: {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator, reference Rng)",
        "config": {**p.summary(), "sample_pairs": npairs, "same_config": npairs == p.pairs},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(p):
    """Bounded sample of the reference CPU path on this host (rank 0, N = 1):
    repeated pair batches until >= 10 s of wall time (<= ~30 s)."""
    threads = os.cpu_count() or 1
    npairs = min(p.pairs, max(1, threads if p.L > 4096 else 4 * threads))
    total_t, total_pairs, reps = 0.0, 0, 0
    while total_t < 10.0 and reps < 64:
        pair0 = (reps * npairs) % p.pairs
        n = min(npairs, p.pairs - pair0)
        dt = reference_run(p, reference_inputs(p, pair0, n), threads)
        total_t += dt
        total_pairs += n
        reps += 1
        if dt > 20.0:
            break
    return {"value": total_pairs * p.L / p.heads / total_t, "unit": "tokens/s", "cores": threads,
            "kind": "reference",
            "sample": f"{reps} batches, {total_pairs} of {p.pairs} (b,h) pairs through oracle/_ref (the "
                      f"reference sources), {total_t:.1f} s wall; tokens = pairs*L/heads",
            "cpu_model": cpu_model()}


# ------------------------------------------------------- rank partitioning
def rank_slice(p, rank: int, world: int) -> tuple[int, int]:
    """This rank's contiguous (b,h)-pair range of the ONE config (strong
    scaling): the config's B*H pairs split over the ranks."""
    from paper_2110_11299_b200.shard import pair_range
    return pair_range(rank, world, p.pairs)


def rank_inputs(p, rank: int, world: int, pinned: bool = False):
    """Seeded inputs of this rank's pairs only (each pair from its own
    substream, so the union over ranks is exactly the N = 1 input)."""
    from paper_2110_11299_b200 import ops
    lo, hi = rank_slice(p, rank, world)
    q, k, v, P = ops.generate(p, pair0=lo, npairs=hi - lo, pinned=pinned)
    return lo, hi, q, k, v, P


def global_checksum(z_local, p, world: int):
    """Per-pair checksums (fp64 sum of Z, max |Z|) of every rank, gathered
    over the process group after timing; returns [sum, max] over the config
    -- identical for every world size."""
    import torch
    from paper_2110_11299_b200.shard import gather_checksums, pair_checksums
    cs = pair_checksums(z_local)
    if world > 1:
        cs = gather_checksums(cs.to(dist_device(cs.device)), p.pairs)
    return [float(cs[:, 0].sum().item()), float(cs[:, 1].max().item())] if cs.shape[0] else [0.0, 0.0]


# ---------------------------------------------------------------- GPU arm
def graph_of(fn, stream):
    """One call of `fn(stream)` captured as a CUDA graph (None if capture fails)."""
    import torch
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn(stream)
        with torch.cuda.stream(stream):
            g.replay()
        stream.synchronize()
        return g
    except Exception as e:  # pragma: no cover - capture unsupported
        print(f"[bench] graph capture failed ({e}); eager launches", file=sys.stderr)
        torch.cuda.synchronize()
        return None


def time_graph(fn, g, stream, reps: int, flush=None) -> float:
    """Mean ms of `reps` replays of graph `g` (or eager `fn`), CUDA events on `stream`."""
    import torch
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    total = 0.0
    for _ in range(reps):
        with torch.cuda.stream(stream):
            if flush is not None:
                flush.fill_(1.0)
            evs[0].record(stream)
            if g is not None:
                g.replay()
            else:
                fn(stream)
            evs[1].record(stream)
        evs[1].synchronize()
        total += evs[0].elapsed_time(evs[1])
    return total / reps


def run_gpu_arm(args, p, rank, local, world):
    import torch
    from paper_2110_11299_b200 import ops

    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    lo, hi, q, k, v, Pm = rank_inputs(p, rank, world, pinned=True)
    P_ = hi - lo
    if P_ == 0:
        raise SystemExit(f"[bench] {p.name} has {p.pairs} (b,h) pairs: fewer than {world} ranks")
    qd, kd, vd, Pd = (t.to(dev) for t in (q, k, v, Pm))
    zd = torch.empty_like(qd)
    zh = torch.empty_like(q).pin_memory()
    stream = torch.cuda.Stream(device=dev)
    pipe = ops.Pipeline(p, pairs=P_, device=dev)
    ph = ops.Phases(p, P_, device=dev)
    in_bytes = q.numel() * q.element_size() * 3
    l2_note = (f"inputs {in_bytes / 1e6:.0f} MB > 126 MB L2 (no flush needed)" if in_bytes > 126e6
               else "L2 flushed between steps (256 MB write)")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if in_bytes <= 126e6 else None

    def step(s):
        if flush is not None:
            flush.fill_(1.0)
        pipe(qd, kd, vd, Pd, out=zd, stream=s)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step(stream)
    stream.synchronize()

    # one step captured as a CUDA graph (replayed per timed step: the same
    # kernels, without host launch gaps); eager launches if capture fails
    graph, per_step = None, None
    if not args.no_graph:
        c0 = ops.launch_counter()
        graph = graph_of(step, stream)
        per_step = ops.launch_counter() - c0

    # ---- device-resident timed region (barrier + sync on both sides, max over ranks)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = ops.launch_counter()
    barrier(world)
    torch.cuda.synchronize(dev)
    with ClockSampler(local % ndev) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                if graph is not None:
                    graph.replay()
                else:
                    step(stream)
            ev1.record(stream)
        ev1.synchronize()
        torch.cuda.synchronize(dev)
    launches = per_step * args.steps if graph is not None else ops.launch_counter() - n0
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms_local, world, dev)
    barrier(world)

    # ---- end to end through the C-ABI with host buffers.  Every step copies
    # its Q/K/V/P in from pinned host memory and Z back out; each step is cut
    # into pair chunks (the public dsa_pipeline on a contiguous pair range)
    # software-pipelined over two device buffer sets, so chunk c+1's H2D and
    # chunk c-1's D2H (separate copy engines / directions) overlap chunk c's
    # kernels and the pipeline's fill / drain shrinks to one chunk.  Timed
    # from the first H2D to the last D2H.
    h2d = in_bytes + Pm.numel() * 4
    d2h = zh.numel() * zh.element_size()
    bufs = [(qd, kd, vd, Pd, zd)] + [tuple(torch.empty_like(t) for t in (qd, kd, vd, Pd, zd))]
    # pair chunks per step: only where the kernels are a sizeable share of the
    # copy time (C1, C4) -- where PCIe dominates (C2, C3) the per-chunk
    # enqueue and event overhead cost more than the shorter drain saves
    copy_ms = (in_bytes + zh.numel() * zh.element_size()) / 50e9 * 1e3
    nch = next(c for c in (4, 2, 1) if P_ % c == 0) if ms > 0.25 * copy_ms else 1
    cp = P_ // nch
    cpipe = ops.Pipeline(p, pairs=cp, device=dev) if nch > 1 else pipe
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev_in = [[torch.cuda.Event() for _ in range(nch)] for _ in range(2)]
    ev_comp = [[torch.cuda.Event() for _ in range(nch)] for _ in range(2)]
    ev_out = [[torch.cuda.Event() for _ in range(nch)] for _ in range(2)]

    def e2e_steps(n):
        for i in range(n):
            b = i & 1
            bq, bk, bv, bp, bz = bufs[b]
            for c in range(nch):
                # whole tensors when unchunked (no per-step view creation)
                cut = (lambda t: t) if nch == 1 else (lambda t, c=c: t[c * cp:(c + 1) * cp])
                with torch.cuda.stream(s_in):
                    if i >= 2:
                        s_in.wait_event(ev_comp[b][c])  # chunk c of buffer b free (step i-2 computed)
                    cut(bq).copy_(cut(q), non_blocking=True)
                    cut(bk).copy_(cut(k), non_blocking=True)
                    cut(bv).copy_(cut(v), non_blocking=True)
                    if c == 0:
                        bp.copy_(Pm, non_blocking=True)
                    ev_in[b][c].record(s_in)
                stream.wait_event(ev_in[b][c])
                if i >= 2:
                    stream.wait_event(ev_out[b][c])  # z chunk drained (step i-2 copied out)
                cpipe(cut(bq), cut(bk), cut(bv), bp, out=cut(bz), stream=stream)
                ev_comp[b][c].record(stream)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_comp[b][c])
                    cut(zh).copy_(cut(bz), non_blocking=True)
                    ev_out[b][c].record(s_out)

    e2e_steps(2)
    torch.cuda.synchronize(dev)
    barrier(world)
    torch.cuda.synchronize(dev)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record(s_in)
    stream.wait_event(t_start)
    s_out.wait_event(t_start)
    e2e_steps(args.steps)
    s_out.wait_event(ev_comp[(args.steps - 1) & 1][nch - 1])
    t_end.record(s_out)
    t_end.synchronize()
    e2e_ms = max_over_ranks(t_start.elapsed_time(t_end) / args.steps, world, dev)
    torch.cuda.synchronize(dev)

    # ---- per-kernel timing for the roofline (CUDA events on the launching
    # stream, graphs replayed like the timed step).  The timed step is
    # predict + the rest of dsa_pipeline (for COLVEC one fused select +
    # attention kernel); the three unfused phases explain it.
    reps = max(3, args.steps)
    g_pred = graph_of(lambda s: ph.predict(qd, kd, Pd, s), stream)
    predict_ms = time_graph(lambda s: ph.predict(qd, kd, Pd, s), g_pred, stream, reps, flush)
    step_ms = time_graph(step, graph, stream, reps) if flush is None else time_graph(
        lambda s: pipe(qd, kd, vd, Pd, out=zd, stream=s), None, stream, reps, flush)
    ph.select(stream)
    stream.synchronize()
    g_sel = graph_of(lambda s: ph.select(s), stream)
    select_ms = time_graph(lambda s: ph.select(s), g_sel, stream, reps, flush)
    g_att = graph_of(lambda s: ph.attend(qd, kd, vd, zd, s), stream)
    attend_ms = time_graph(lambda s: ph.attend(qd, kd, vd, zd, s), g_att, stream, reps, flush)
    pipe(qd, kd, vd, Pd, out=zd, stream=stream)  # Z of the timed path, for the checksum
    stream.synchronize()

    # ---- checksums over the process group after timing (not on the hot path)
    csum = global_checksum(zd, p, world)

    if rank != 0:
        return
    peaks, peak_src = load_peaks()
    L, d, k_, e = p.L, p.d, p.k, (2 if p.dtype == "bf16" else 4)
    pairs = P_
    cnt = ops.counters(p, ph.mask, pairs, stream=stream)
    nnz = cnt["nnz"]
    causal = p.mask_mode == "threshold" and p.causal
    score_flops = (L * (L + 1) if causal else 2 * L * L) * k_ * pairs
    # algorithmic work per launch of each phase over this rank's pairs
    work = {
        "predict": {"bound": "hbm", "amount": (2 * L * d * e + 2 * L * k_ * 2) * pairs + d * k_ * 4,
                    "unit": "GB/s", "scale": 1e9},
        "select": {"bound": "tensor", "amount": score_flops, "unit": "TFLOP/s", "scale": 1e12},
        "attention": {"bound": "hbm", "amount": 4 * L * d * e * pairs, "unit": "GB/s", "scale": 1e9},
    }
    if p.mask_mode == "block":
        # C3: the selection ranks pooled block scores (no L^2 score GEMM): it
        # streams the levels and writes the block lists -> HBM; 32x32 blocks
        # put the attention near the ridge -> tensor
        nbk = -(-L // p.block)
        work["select"] = {"bound": "hbm", "amount": (2 * L * k_ * 2 + nbk * p.keep * 4) * pairs,
                          "unit": "GB/s", "scale": 1e9}
        work["attention"] = {"bound": "tensor", "amount": 4 * nnz * d, "unit": "TFLOP/s", "scale": 1e12}
    phase_ms = {"predict": predict_ms, "select": select_ms, "attention": attend_ms}
    fused = p.mask_mode == "colvec" and ops.fused_pipeline(p, pairs)
    rest_ms = max(step_ms - predict_ms, 1e-6)
    if fused:
        # the timed step's dominant kernel: colvec_tc_kernel<.., FUSED> =
        # score GEMM + pooling + selection + SDDMM/softmax/SpMM
        dom = "select+attention (fused colvec_tc_kernel)"
        w = {"bound": "tensor", "amount": score_flops + 4 * nnz * d, "unit": "TFLOP/s", "scale": 1e12}
        dom_ms = rest_ms
    else:
        dom = max(phase_ms, key=phase_ms.get)
        w = work[dom]
        dom_ms = phase_ms[dom]
    achieved = w["amount"] / (dom_ms * 1e-3) / w["scale"]
    peak = peaks["hbm_gbs"] if w["bound"] == "hbm" else peaks["bf16_tflops"]
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(f"{p.name}:{'fused' if fused else dom}")
    phases = {}
    for kx, ms_k in phase_ms.items():
        wk = work[kx]
        a_k = wk["amount"] / (ms_k * 1e-3) / wk["scale"]
        pk = peaks["hbm_gbs"] if wk["bound"] == "hbm" else peaks["bf16_tflops"]
        phases[kx] = {"ms": ms_k, "bound": wk["bound"], "achieved": a_k, "unit": wk["unit"], "frac": a_k / pk}
    if fused:
        phases["fused_select_attention"] = {"ms": rest_ms, "bound": "tensor", "achieved": achieved,
                                            "unit": "TFLOP/s", "frac": achieved / peak,
                                            "note": "timed step minus predict (both CUDA-event timed)"}
    # explanatory counters: candidates scored per second, and the
    # K/V row bytes the attention gathers (reuse = query rows sharing a gather)
    cand = (L * (L + 1) // 2 if causal else L * L) * pairs
    phases["select"]["candidates_per_s"] = cand / (select_ms * 1e-3)
    reuse = {"colvec": p.vec_v, "block": p.block}.get(p.mask_mode, 1)
    phases["attention"]["gathered_GBps"] = 2 * nnz * d * e / reuse / (attend_ms * 1e-3) / 1e9
    phases["attention"]["gather_reuse"] = reuse
    # the reference's dataflow cost model (P/src/dataflow.cpp:10-62, SURVEY
    # 8(f)4) on this mask: operand fetches of row-parallel bands of 8 rows,
    # in kept order and reordered (the band column union) -- the reuse a
    # query-tile union staging could exploit (built, slower)
    try:
        df = {}
        for sched in ("row_parallel", "row_parallel_reordered"):
            f, _ = ops.dataflow_trace(p, ph.mask, pairs, sched, 8, stream=stream)
            df[sched] = nnz / max(int(f.sum()), 1)
        phases["attention"]["dataflow_reuse_band8"] = df
    except Exception as ex:  # noqa: BLE001 -- explanatory only (L > 65536)
        phases["attention"]["dataflow_reuse_band8"] = {"unavailable": str(ex)[:80]}
    tokens = p.tokens  # the whole config: every rank's pairs
    value = tokens / (ms * 1e-3)
    adjacent = None
    if not args.no_adjacent:
        adjacent = {"project_qkv": time_project_qkv(p, peaks["bf16_tflops"])}
        if world == 1:
            adjacent["layer_e2e"] = time_layer_e2e(p, steps=max(3, min(args.steps, 10)))
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(p)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16" if p.dtype == "bf16" else "f32",
        "data": "synthetic (seeded BASELINE generator, SURVEY 8.0)",
        "config": {**p.summary(), "pairs_per_gpu": pairs, "parallelism": f"(b,h)-pairs /{world}",
                   "launch": "cuda graph per step" if graph is not None else "eager",
                   "l2": l2_note, **({"oversubscribed_gpus": True} if world > ndev else {})},
        "e2e": {"value": tokens / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "pair_chunks_per_step": nch},
        "roofline": {"kernel": dom, "bound": w["bound"], "achieved": achieved, "peak": peak,
                     "unit": w["unit"], "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src,
                     "note": ROOFLINE_NOTES.get("fused" if fused else
                                                (dom if not (dom == "attention" and w["bound"] == "tensor")
                                                 else "attention_block"), "")},
        "phases": phases,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "counters": {"nnz": nnz, "sddmm_mults": cnt["sddmm_mults"], "spmm_mults": cnt["spmm_mults"],
                     "softmax_exps": cnt["softmax_exps"]},
        "checksum": csum,
    }
    if adjacent:
        line["adjacent"] = adjacent
    print(json.dumps(line), flush=True)


# what bounds each phase beyond its nominal roofline
ROOFLINE_NOTES = {
    "fused": "achieved = (2*L^2*k score-GEMM + 4*nnz*d attention) flops over the fused kernel's time "
             "(timed step minus predict); the kernel is bound by the per-score integer work of pooling and "
             "exact selection (issue-bound), not by the tensor pipe -- DESIGN.md 4",
    "select": "achieved = the 2*L^2*k score-GEMM flops (K = k = 16/32 per MMA) over the select time; the "
              "kernel is bound by the per-score integer selection work that follows each MMA (issue-bound, "
              "ncu IPC ~2.3-2.6), not by the tensor pipe, so this fraction is small by construction -- "
              "phases.select.candidates_per_s is the throughput that matters",
    "attention": "bytes = compulsory Q/K/V/Z traffic; the kernels are bound by the row gathers "
                 "(phases.attention.gathered_GBps, served from L2/L1)",
    "attention_block": "flops = 4*nnz*d (32x32 blocks: each kept block's K/V rows staged once in shared "
                       "memory for the 32 queries of its block row, mma.sync m16n8k16)",
    "predict": "bytes = Q/K read once + levels written",
}


def time_layer_e2e(p, steps=5):
    """Layer-level end to end (adjacent, not `value`/`e2e`): the caller hands
    over the layer input X (pinned host, bf16) instead of Q/K/V; per step X
    goes H2D, dsa_project_qkv makes every head's Q/K/V on the device, the
    DSA pipeline runs and Z comes back D2H.  Pipelined over two buffer sets
    like `e2e`; weights (packed W, P) are device-resident parameters."""
    import torch
    from paper_2110_11299_b200 import ops
    sh = p.shape
    dm, heads, dk, dv = sh["d"], p.heads, sh["d_k"], sh["d_v"]
    if dk != p.d or dv != p.d or p.dtype != "bf16":
        return None
    dev = torch.device("cuda")
    x = torch.randn(p.batch, p.L, dm).to(torch.bfloat16).pin_memory()
    w = (torch.randn(heads * (2 * dk + dv), dm, device=dev) / dm ** 0.5).to(torch.bfloat16)
    _, _, _, Pm = ops.generate(p.replace(batch=1, heads=1), npairs=1)
    Pd = Pm.to(dev)
    pipe = ops.Pipeline(p, device=dev)
    zh = torch.empty(p.pairs, p.L, p.d, dtype=torch.bfloat16).pin_memory()
    bufs = [(torch.empty_like(x, device=dev),
             ops.project_qkv(torch.empty_like(x, device=dev), w, heads, dk, dv)[:3],
             torch.empty(p.pairs, p.L, p.d, dtype=torch.bfloat16, device=dev)) for _ in range(2)]
    stream, s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def run(n):
        for i in range(n):
            b = i & 1
            xd, (qd, kd, vd), zd = bufs[b]
            with torch.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(ev_comp[b])
                xd.copy_(x, non_blocking=True)
                ev_in[b].record(s_in)
            stream.wait_event(ev_in[b])
            if i >= 2:
                stream.wait_event(ev_out[b])
            ops.project_qkv(xd, w, heads, dk, dv, stream=stream, out=(qd, kd, vd, None))
            pipe(qd, kd, vd, Pd, out=zd, stream=stream)
            ev_comp[b].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_comp[b])
                zh.copy_(zd, non_blocking=True)
                ev_out[b].record(s_out)

    run(2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(steps)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    return {"value": p.tokens / (ms * 1e-3), "unit": "tokens/s", "ms_per_step": ms, "steps": steps,
            "h2d_bytes_per_step": x.numel() * 2, "d2h_bytes_per_step": zh.numel() * 2,
            "note": "adjacent, NOT the metric: from the layer input X (d_model = %d) instead of Q/K/V -- "
                    "H2D X, dsa_project_qkv, dsa_pipeline, D2H Z per step (wall clock over the pipelined "
                    "steps); only X crosses PCIe" % dm}


def time_project_qkv(p, peak_tflops, reps=10):
    """The step before the path, outside the timed region and
    not part of `value`: dsa_project_qkv on this config's layer shape
    (d_model, heads, d_k, d_v from the preset `shape`, npred = k), CUDA
    events on the launching stream."""
    import torch
    from paper_2110_11299_b200 import ops
    sh = p.shape
    dm, heads, dk, dv = sh["d"], p.heads, sh["d_k"], sh["d_v"]
    batch = max(1, min(p.batch, 131072 // p.L))
    M, N = batch * p.L, heads * (2 * dk + dv) + p.k
    x = torch.randn(batch, p.L, dm, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, dm, device="cuda") / dm ** 0.5).to(torch.bfloat16)
    out = (torch.empty(batch * heads, p.L, dk, dtype=torch.bfloat16, device="cuda"),
           torch.empty(batch * heads, p.L, dk, dtype=torch.bfloat16, device="cuda"),
           torch.empty(batch * heads, p.L, dv, dtype=torch.bfloat16, device="cuda"),
           torch.empty(batch, p.L, p.k, dtype=torch.float32, device="cuda"))
    st = torch.cuda.current_stream()
    for _ in range(3):
        ops.project_qkv(x, w, heads, dk, dv, p.k, stream=st, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        ops.project_qkv(x, w, heads, dk, dv, p.k, stream=st, out=out)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 2.0 * M * N * dm / (ms * 1e-3) / 1e12
    return {"kernel": "qkv_gemm_kernel (tcgen05, TMA)", "M": M, "N": N, "K": dm, "ms": ms, "bound": "tensor",
            "achieved": tf, "unit": "TFLOP/s", "peak": peak_tflops, "frac": tf / peak_tflops,
            "note": "X W^T for every head's Q/K/V + predictor input R = X P (project_qkv, "
                    "P/src/attention.cpp:36-46); random weights; not part of value"}


def spawn_ranks(n: int) -> None:
    """`--gpus N` outside torchrun: re-launch this command as N ranks (one
    process per GPU) under torch.distributed.run on 127.0.0.1."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2_vector")
    ap.add_argument("--ref-pairs", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-adjacent", action="store_true", help="skip the project_qkv GEMM measurement")
    ap.add_argument("--no-graph", action="store_true", help="eager launches in the timed region")
    args = ap.parse_args()
    from paper_2110_11299_b200 import load_preset

    p = load_preset(args.config)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        spawn_ranks(args.gpus)
    if args.impl == "reference":
        # CPU only: rank 0 runs and prints, the other ranks exit 0 without
        # work -- no process group (no collective is needed)
        run_reference_arm(args, p, int(os.environ.get("RANK", "0")), max(args.gpus, int(os.environ.get("WORLD_SIZE", "1"))))
        return
    rank, local, world = dist_setup()
    try:
        run_gpu_arm(args, p, rank, local, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
