"""Benchmark: re-ranking throughput of the sparse cross-encoder on B200.

Metric (BASELINE.json): query-doc pairs/sec at 4096 tok w=4 (1/2/4/8 B200);
attn kernel HBM GB/s % peak.

Workload (BASELINE.json configs[2], the config the metric is quoted on):
ELECTRA-base sparse cross-encoder (12 layers, h=768, 12 heads, ff=3072,
vocab 30522, random-init weights with the reference's init_weights draw
order), asymmetric pattern w=4, documents of 4096 tokens = q10 + d4086 + 3
specials = s 4099 (T/test_bench.py:66-70), packed varlen batch of
`--pairs-per-gpu` pairs per GPU, bf16 GEMMs/attention/residual stream (fp32 LayerNorm
statistics).  A "step" = one forward of the whole per-GPU batch (12 layers +
scores) + one NCCL all-gather of the fp32 scores.

  python bench.py [--gpus N --steps K --warmup W]            # our arm
  python bench.py --impl reference [...]                      # CPU oracle arm
  torchrun --nproc-per-node N bench.py --gpus N ...           # N > 1

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "query-doc pairs/sec at 4096 tok w=4 (1/2/4/8 B200); attn kernel HBM GB/s % peak"
ELECTRA = dict(layers=12, embed_dim=768, heads=12, ff_dim=3072, vocab_size=30522, pattern="sparse", window=4)
QUERY_LEN = 10


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return d["hbm_gbs"], d["bf16_tflops"], d["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def workload(args):
    """(encoder config, doc_len, s): documents (configs[2], s=4099) or passages (configs[1], s=177)."""
    doc_len = args.doc_len
    s = QUERY_LEN + doc_len + 3
    return dict(ELECTRA, max_positions=max(s, 512)), doc_len, s


def workload_name(doc_len, s):
    if doc_len <= 512:
        return (f"ELECTRA-base sparse cross-encoder, passages {QUERY_LEN + doc_len} tok (q{QUERY_LEN}+p{doc_len}, "
                f"s={s}), w=4 asymmetric, bf16 (BASELINE configs[1])")
    return (f"ELECTRA-base sparse cross-encoder, documents {QUERY_LEN + doc_len} tok (q{QUERY_LEN}+d{doc_len}, "
            f"s={s}), w=4 asymmetric, packed batch (BASELINE configs[2])")


def make_batch(P, cfg, doc_len, pairs, rank, seed=0, varlen=False):
    """Synthetic pairs (query q, candidate i) with ids from default_rng((seed, q, i))."""
    seqs = []
    rng = np.random.default_rng((seed, 7919, rank))
    for i in range(pairs):
        q = rank * 1000 + i // 100
        qids = np.random.default_rng((seed, q)).integers(3, cfg["vocab_size"], size=QUERY_LEN)
        n = int(rng.integers(54, doc_len + 1)) if varlen else doc_len
        dids = np.random.default_rng((seed, q, i % 100)).integers(3, cfg["vocab_size"], size=n)
        seqs.append(P.assemble_input(qids, dids, cfg["max_positions"]))
    return P.PackedBatch.from_sequences(seqs)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        under = [x for x in sm if mx and x > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(under) if under else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference): the ONLY place
# bench.py executes oracle/, as the timed CPU baseline.
# ---------------------------------------------------------------------------

def cpu_oracle_pair_times(cfg, doc_len, reps, budget_s=None):
    """Seconds per whole pair on the CPU oracle: embed + 12 layers + score head of ONE (q10, d)
    pair (R/encoder.py:475-509 restated in oracle/), f32 numpy on all host cores.  Stops after
    ``budget_s`` seconds (at least one timed pair)."""
    from oracle import sparsecross_oracle as O

    wt = O.init_weights(dict(cfg), 0, np.float32)
    ids, spans = O.gen_random_ids(0, QUERY_LEN, doc_len, 1, cfg["vocab_size"])
    times = []
    t_start = time.perf_counter()
    for _ in range(reps):
        t0 = time.perf_counter()
        O.score(ids, spans, dict(cfg), wt)
        times.append(time.perf_counter() - t0)
        if budget_s and time.perf_counter() - t_start > budget_s:
            break
    return times


def cpu_threads():
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
        if os.environ.get(v, "").isdigit():
            return int(os.environ[v])
    return os.cpu_count() or 1


def bench_config(args, world, n, s, doc_len, use_graph, total_tokens):
    """The line's ``config`` (both arms print the same dict for the same flags)."""
    return {"workload": workload_name(doc_len, s), "cuda_graph": bool(use_graph),
            "prune_last_layer": bool(args.prune_last_layer), "pairs_per_gpu": n, "global_batch": n * world,
            "seq_len": s, "doc_len": doc_len, "query_len": QUERY_LEN, "varlen": bool(args.varlen), "pattern": "sparse",
            "window": 4, "layers": 12, "hidden": 768, "heads": 12, "ff": 3072, "parallelism": f"dp{world}",
            "l2": f"inputs larger than L2 (qkv activations {total_tokens * 2304 * 2 / 1e9:.2f} GB per layer)"}


def run_reference(args):
    """The reference arm: the CPU restatement of the reference's CrossEncoder.score (f32 numpy,
    all host cores), one whole (q10, d4086) pair per step -- the same workload, config and metric
    as the GPU arm, bounded so the run ends within a few minutes (--ref-budget seconds)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, doc_len, s = workload(args)
    cpu_oracle_pair_times(cfg, doc_len, 1)  # warm-up: page in the weights (one pair)
    times = cpu_oracle_pair_times(cfg, doc_len, args.steps, budget_s=args.ref_budget)
    t_pair = statistics.median(times)
    value = 1.0 / t_pair
    sample = (f"{len(times)} whole pairs at s={s} (q{QUERY_LEN}+d{doc_len}): embed + {cfg['layers']} layers + score "
              f"head, f32 numpy oracle port of R/encoder.py:475-509 (pinned to reference goldens); pairs/s = "
              f"1 / median pair time ({t_pair:.2f} s); timed steps capped by a {args.ref_budget:.0f} s budget")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": 1, "ms_per_step": t_pair * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generator ids, seed 0)",
        "config": bench_config(args, int(os.environ.get("WORLD_SIZE", "1")), args.pairs_per_gpu, s, doc_len,
                               args.graph == "on" or (args.graph == "auto" and doc_len <= 512),
                               args.pairs_per_gpu * s),
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cpu_threads(), "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# Parity of the bench's own output, and the variant workloads (C2 passages,
# varlen documents, the C4 attention sweep) recorded beside the headline.
# ---------------------------------------------------------------------------

GOLDEN = os.path.join(ROOT, "tests", "golden")
BF16_TOL = 2e-2


def rank_order(scores):
    """R/evaluation.py:194-201: stable sort by (-score, candidate position)."""
    return sorted(range(len(scores)), key=lambda j: (-float(scores[j]), j))


def parity(scores, ref, tol, source):
    """Max |score - reference| of the bench's own first len(ref) pairs (which ARE the golden pairs:
    ids from default_rng((0, 0, j))), ranking identity and flips beyond 2 x tol."""
    k = min(len(scores), len(ref))
    got, ref = np.asarray(scores[:k], np.float64), np.asarray(ref[:k], np.float64)
    ro, pos = rank_order(ref), {c: i for i, c in enumerate(rank_order(got))}
    flips = sum(1 for a in range(k) for b in range(a + 1, k)
                if pos[ro[a]] > pos[ro[b]] and abs(ref[ro[a]] - ref[ro[b]]) > 2 * tol)
    return {"max_abs_err": float(np.abs(got - ref).max()), "n": k, "tol": tol,
            "ranking_identical": rank_order(got) == ro, "flips_beyond_2tol": flips, "reference": source}


def headline_parity(scores_np, doc_len, varlen):
    try:
        if varlen:
            return None
        if doc_len == 4086:
            ref = np.load(os.path.join(GOLDEN, "ranking.npz"))["scores"]
            src = "tests/golden/ranking.npz: unmodified reference CrossEncoder.score (f32) on the same pairs"
        elif doc_len == 164:
            ref = np.load(os.path.join(GOLDEN, "encoder.npz"))["electra_passage_scores"]
            src = "tests/golden/encoder.npz:electra_passage_scores (unmodified reference, f32)"
        else:
            return None
        return parity(scores_np, ref, BF16_TOL, src)
    except FileNotFoundError:
        return None


def attn_kvalid(pattern, lens, qds=False):
    """Valid (row, key) pairs of one sequence under ``pattern`` (SURVEY §8d K_valid): full links
    count rows x target length, windowed doc->doc links the in-range band slots."""
    gl = dict(zip(("cls", "query", "doc"), lens))
    total = 0
    for src, tl in pattern.targets.items():
        for tgt, w in tl:
            if w == math.inf:
                total += gl[src] * gl[tgt]
            else:
                n = gl[src]
                r = np.arange(n)
                total += int((np.minimum(n - 1, r + w) - np.maximum(0, r - w) + 1).sum())
    return total


def attention_sweep(P, dev, peaks_, nseq=64, doc=4086, H=12, d=64, reps=10,
                    windows=(("sparse", 1), ("sparse", 4), ("sparse", 16), ("sparse", 64), ("sparse", 256),
                             ("sparse", math.inf), ("full", math.inf))):
    """C4 (BASELINE configs[3]): sc_attn_fwd alone at s=4099 over a packed batch of ``nseq``
    sequences, bf16 Q/K/V ~ N(0,1); per window: time, algorithmic GB/s (4*s*h*2 B per sequence-layer)
    and TFLOP/s (4*d*H*K_valid), each against its measured peak; the binding one is ``bound``."""
    import torch

    hbm, tf_burst = peaks_[0], peaks_[1]
    s = QUERY_LEN + doc + 3
    T = s * nseq
    lay = P.PackedLayout.from_lengths([s] * nseq, [QUERY_LEN + 1] * nseq, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    qkv = torch.randn((T, 3 * H * d), device=dev, generator=g).to(torch.bfloat16)
    out = torch.empty((T, H * d), device=dev, dtype=torch.bfloat16)
    st = torch.cuda.current_stream(dev)
    res = []
    for name, w in windows:
        pat = P.make_pattern(name, w)
        f = lambda: P.attend_packed(qkv[:, :H * d], qkv[:, H * d:2 * H * d], qkv[:, 2 * H * d:], lay, pat, H,
                                    out=out, check=False)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            f()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        byts = 4 * T * H * d * 2
        flops = 4 * d * H * attn_kvalid(pat, (1, QUERY_LEN + 1, doc + 1)) * nseq
        gbs, tfs = byts / ms / 1e6, flops / ms / 1e9
        bound = "hbm" if flops / byts < tf_burst * 1e12 / (hbm * 1e9) else "tensor"
        res.append({"pattern": name, "window": "inf" if w == math.inf else int(w), "ms": round(ms, 4),
                    "us_per_seq_layer": round(ms * 1e3 / nseq, 2), "GB/s": round(gbs, 1),
                    "frac_hbm": round(gbs / hbm, 3), "TFLOP/s": round(tfs, 1), "frac_tensor": round(tfs / tf_burst, 3),
                    "bound": bound, "frac_of_bound": round(gbs / hbm if bound == "hbm" else tfs / tf_burst, 3)})
    return {"workload": f"sc_attn_fwd alone, {nseq} x s={s} packed, H={H}, d={d}, bf16, AUTO kernel choice",
            "peaks": {"hbm_GBs": hbm, "bf16_TFLOPs_burst": tf_burst}, "reps": reps, "points": res}


def timed_scores(fn, steps, stream):
    """CUDA-event time (ms) of ``steps`` back-to-back calls of fn after 3 warm-ups."""
    import torch

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def passages_variant(P, dev, steps, pairs=1024):
    """C2 (BASELINE configs[1]): 1024 passages (q10 + p164, s=177) per step as one CUDA graph."""
    import torch
    from paper_2312_17649_b200.encoder import GraphedScorer

    cfg = dict(ELECTRA, max_positions=512)
    model = P.CrossEncoder(P.EncoderConfig(**cfg, precision="bf16"), seed=0, device=dev)
    batch = make_batch(P, cfg, 164, pairs, 0)
    gs = GraphedScorer(model, batch)
    ids_dev = torch.from_numpy(batch.ids).to(dev)
    ms = timed_scores(lambda: gs(ids_dev), steps, torch.cuda.current_stream(dev))
    sc = gs(ids_dev).cpu().numpy()
    return {"value": pairs * steps / (ms / 1e3), "unit": "pairs/s", "ms_per_step": ms / steps, "steps": steps,
            "pairs_per_step": pairs, "seq_len": 177, "cuda_graph": True, "dtype": "bf16",
            "parity": headline_parity(sc, 164, False)}


def fp32_variant(P, dev, steps, pairs=32):
    """Ranking-exact fp32 (north-star "identical per-query rankings"): the same documents in fp32,
    projections as split-fp16 / split-bf16 tensor-core products (fp32_gemm="f16x3" / "bf16x6") vs
    cuBLAS SGEMM; parity of each against the reference golden of these exact pairs."""
    import torch

    cfg = dict(ELECTRA, max_positions=4099)
    batch = make_batch(P, cfg, 4086, pairs, 0)
    out = {}
    for mode, nsteps in (("f16x3", steps), ("bf16x6", steps), ("sgemm", 2)):
        model = P.CrossEncoder(P.EncoderConfig(**cfg, precision="f32"), seed=0, device=dev, fp32_gemm=mode)
        layout = model.make_layout(batch)
        ids = torch.from_numpy(batch.ids).to(dev)
        fn = lambda: model.scores_from_hidden(model.encode_packed(ids, layout), layout)
        ms = timed_scores(fn, nsteps, torch.cuda.current_stream(dev))
        sc = fn().cpu().numpy()
        par = headline_parity(sc, 4086, False)
        if par is not None:
            par["tol"] = 2e-6  # tests/test_gpu_headline.py; cuBLAS SGEMM itself lands at ~1.5e-6
            par["flips_beyond_2tol"] = None
        out[mode] = {"value": pairs * nsteps / (ms / 1e3), "unit": "pairs/s", "ms_per_step": ms / nsteps,
                     "steps": nsteps, "pairs_per_step": pairs, "dtype": "f32", "parity": par}
        del model
        torch.cuda.empty_cache()
    out["speedup_vs_sgemm"] = {m: out[m]["value"] / out["sgemm"]["value"] for m in ("f16x3", "bf16x6")}
    return out


def varlen_variant(P, dev, model, steps, pairs=64):
    """Documents with lengths ~ U{54..4086}, packed varlen, same model."""
    import torch

    cfg = dict(ELECTRA, max_positions=4099)
    batch = make_batch(P, cfg, 4086, pairs, 0, varlen=True)
    layout = model.make_layout(batch)
    ids = torch.from_numpy(batch.ids).to(dev)
    fn = lambda: model.scores_from_hidden(model.encode_packed(ids, layout), layout)
    ms = timed_scores(fn, steps, torch.cuda.current_stream(dev))
    return {"value": pairs * steps / (ms / 1e3), "unit": "pairs/s", "ms_per_step": ms / steps, "steps": steps,
            "pairs_per_step": pairs, "tokens_per_step": int(layout.total_tokens), "dtype": "bf16"}


# ---------------------------------------------------------------------------
# GPU arm.
# ---------------------------------------------------------------------------

def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2312_17649_b200 as P
    from paper_2312_17649_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    gloo = args.dist_backend == "gloo"
    # gloo (test harness only): several ranks may share one GPU; collectives run on host copies
    local = local % torch.cuda.device_count() if gloo else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    _lib.load()
    hbm_peak, tf_burst, tf_sus, peak_kind = peaks()
    cfg, doc_len, s = workload(args)
    ecfg = P.EncoderConfig(**cfg, precision="bf16")
    model = P.CrossEncoder(ecfg, seed=0, device=dev, prune_last_layer=args.prune_last_layer)
    batch = make_batch(P, cfg, doc_len, args.pairs_per_gpu, rank, varlen=args.varlen)
    layout = model.make_layout(batch)
    ids_host = torch.from_numpy(batch.ids).pin_memory()
    ids_dev = ids_host.to(dev)
    n = batch.nseq
    gathered = torch.empty(n * world, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def gather(scores):
        if world > 1 and gloo:
            parts = [torch.empty_like(scores, device="cpu") for _ in range(world)]
            dist.all_gather(parts, scores.cpu())
            return torch.cat(parts).to(dev)
        if world > 1:
            dist.all_gather_into_tensor(gathered, scores)
            return gathered
        return scores

    def reduce_max(t):  # device scalar -> max over ranks
        if world > 1 and gloo:
            c = t.cpu()
            dist.all_reduce(c, op=dist.ReduceOp.MAX)
            return c
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t

    attn_events = []

    def hook(tag):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        attn_events.append(ev)

    use_graph = args.graph == "on" or (args.graph == "auto" and doc_len <= 512)
    graphed = None
    if use_graph:
        from paper_2312_17649_b200.encoder import GraphedScorer

        graphed = GraphedScorer(model, batch)

    def device_step(h=None):
        if graphed is not None:
            return gather(graphed(ids_dev))
        x = model.encode_packed(ids_dev, layout, attn_hook=h, cls_only=model.prune_last_layer)
        return gather(model.scores_from_hidden(x, layout))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- value: device-resident inputs -------------------------------------
    for _ in range(args.warmup):
        device_step()
    barrier()
    launches0 = _lib.kernel_launches()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            device_step(hook)
        e1.record(stream)
        barrier()
    launches = _lib.kernel_launches() - launches0
    if graphed is not None:  # replayed kernels: captured count x replays
        launches += graphed.kernels_per_replay * args.steps
    ms = e0.elapsed_time(e1)
    attn_ms = [attn_events[i].elapsed_time(attn_events[i + 1]) for i in range(0, len(attn_events), 2)]
    ms_max = float(reduce_max(torch.tensor([ms], device=dev)).item())
    pairs_total = n * world * args.steps
    value = pairs_total / (ms_max / 1e3)

    # ---- e2e: public API from pinned host ids, scores back to the host ------
    host_scores = torch.empty(n * world, dtype=torch.float32).pin_memory()

    def e2e_step():
        if graphed is not None:  # GraphedScorer.__call__: H2D of the pinned ids + replay
            sc = gather(graphed(ids_host))
        else:
            ids = ids_host.to(dev, non_blocking=True)
            lay = model.make_layout(batch)
            x = model.encode_packed(ids, lay, cls_only=model.prune_last_layer)
            sc = gather(model.scores_from_hidden(x, lay))
        host_scores.copy_(sc, non_blocking=True)
        return sc

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    e2e_steps = args.steps
    for _ in range(e2e_steps):
        e2e_step()
    f1.record(stream)
    barrier()
    te = reduce_max(torch.tensor([f0.elapsed_time(f1)], device=dev))
    e2e_value = n * world * e2e_steps / (float(te.item()) / 1e3)

    # ---- parity of this run's own scores (outside the timed regions) ----
    own = device_step().cpu().numpy()[:n]  # every rank (the step's gather is a collective)
    par = headline_parity(own, doc_len, args.varlen) if rank == 0 else None

    # ---- variant: last layer on the [CLS] rows only (opt-in serving mode) ----
    variants = {}
    if not args.prune_last_layer and graphed is None:
        model.prune_last_layer = True
        for _ in range(2):
            device_step()
        barrier()
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        vsteps = max(3, args.steps // 4)
        v0.record(stream)
        for _ in range(vsteps):
            device_step()
        v1.record(stream)
        barrier()
        tv = reduce_max(torch.tensor([v0.elapsed_time(v1)], device=dev))
        model.prune_last_layer = False
        variants["prune_last_layer"] = {
            "value": n * world * vsteps / (float(tv.item()) / 1e3), "unit": "pairs/s", "steps": vsteps,
            "note": "CrossEncoder(prune_last_layer=True): last layer past K/V on the [CLS] rows only (the score "
                    "reads x[:,0], R/encoder.py:506); same scores, not the headline"}
    if world == 1 and not args.no_variants and doc_len == 4086 and not args.varlen:
        # the kernel-alone sweeps first (before the GEMM-heavy variants), clocks sampled during each
        with ClockSampler(local) as sclk:
            variants["attention_sweep"] = attention_sweep(P, dev, (hbm_peak, tf_burst))
        variants["attention_sweep"]["clocks"] = sclk.summary()
        with ClockSampler(local) as sclk:
            variants["attention_sweep_d32"] = attention_sweep(  # MiniLM-L6-H384 heads: 12 x d=32
                P, dev, (hbm_peak, tf_burst), d=32, windows=(("sparse", 4), ("sparse", 64), ("sparse", 256)))
        variants["attention_sweep_d32"]["clocks"] = sclk.summary()
        variants["varlen_documents"] = varlen_variant(P, dev, model, max(3, args.steps // 2))
        variants["passages"] = passages_variant(P, dev, args.steps)
        variants["fp32_ranking_exact"] = fp32_variant(P, dev, max(3, args.steps // 4))

    # ---- roofline of the attention kernel (sc_attn_fwd, band + head-row pass) ----
    attn_bytes = 4 * layout.total_tokens * cfg["embed_dim"] * 2  # Q,K,V read + O write, bf16
    def attn_standalone_ms(reps=20):
        """sc_attn_fwd alone on this step's layout and shapes, CUDA events on the launching stream."""
        h, H = cfg["embed_dim"], cfg["heads"]
        qkv = torch.randn((layout.total_tokens, 3 * h), device=dev).to(torch.bfloat16)
        out = torch.empty((layout.total_tokens, h), device=dev, dtype=torch.bfloat16)
        pat = P.make_pattern(cfg["pattern"], cfg["window"])
        run = lambda: P.attend_packed(qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:], layout, pat, H, out=out, check=False)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        # back-to-back launches between two events (a per-launch event pair would
        # also time the host-side launch latency of an idle GPU); 5 trials
        trials = []
        for _ in range(5):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(reps):
                run()
            a1.record(stream)
            torch.cuda.synchronize()
            trials.append(a0.elapsed_time(a1) / reps)
        return trials

    alone_ms = attn_standalone_ms()
    attn_where = "in-step CUDA events around every sc_attn_fwd launch of the timed region"
    if not attn_ms:  # graph replay: no per-launch events inside the graph
        attn_ms = alone_ms
        attn_where = "standalone CUDA-event timing of sc_attn_fwd on this step's layout (step runs as a CUDA graph)"
    attn_avg_ms = statistics.mean(attn_ms)
    alone_gbs = attn_bytes / (statistics.median(alone_ms) / 1e3) / 1e9
    achieved = attn_bytes / (attn_avg_ms / 1e3) / 1e9
    gemm_flops_step = 2 * layout.total_tokens * cfg["layers"] * (4 * cfg["embed_dim"] ** 2 + 2 * cfg["embed_dim"] * cfg["ff_dim"])
    traffic = None
    prof = os.path.join(ROOT, "profiles", "attn_band_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as fh:
                tr = json.load(fh)
            if tr.get("seq_len") == s:
                traffic = tr["dram_bytes_per_launch_per_seq"] * n
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        times = cpu_oracle_pair_times(cfg, doc_len, reps=50, budget_s=args.cpu_budget)
        tp = statistics.median(times)
        cpu = {"value": 1.0 / tp, "unit": "pairs/s", "cores": cpu_threads(), "kind": "port",
               "sample": f"{len(times)} whole pairs at s={s} (embed + {cfg['layers']} layers + score head, f32 numpy "
                         f"oracle port of R/encoder.py:475-509), median {tp:.2f} s/pair"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: reference-generator token ids (default_rng((seed,q,i))), random-init ELECTRA-base weights",
            "config": bench_config(args, world, n, s, doc_len, use_graph, layout.total_tokens),
            "roofline": {"bound": "hbm", "kernel": "sc_attn_fwd (band_attn_kernel + head-row combine)",
                         "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                         "peak_kind": peak_kind, "traffic": traffic,
                         "algorithmic_bytes_per_launch": attn_bytes, "avg_launch_ms": attn_avg_ms,
                         "launches": len(attn_ms), "frac_of_8TBs": achieved / 8000.0,
                         "share_of_step": (sum(attn_ms) / ms) if not use_graph else None,
                         "timing": attn_where,
                         "standalone": {"achieved": alone_gbs, "frac": alone_gbs / hbm_peak,
                                        "median_ms": statistics.median(alone_ms),
                                        "note": "same launch, 20 back-to-back launches between CUDA events, median of 5 trials (GPU not power-capped by the GEMMs)"}},
            "step_roofline": {"bound": "tensor", "achieved": gemm_flops_step / (ms_max / args.steps / 1e3) / 1e12,
                              "peak": tf_sus, "unit": "TFLOP/s", "note": "GEMM FLOPs per step / step time vs sustained bf16"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": int(batch.ids.nbytes),
                    "d2h_bytes_per_step": int(host_scores.numel() * 4), "steps": e2e_steps,
                    "path": ("GraphedScorer.__call__ from pinned host ids (captured layout reused: same shape)"
                             if graphed is not None else
                             "CrossEncoder.make_layout (K1 index build) + encode_packed + scores_from_hidden from "
                             "pinned host ids, scores copied back"),
                    "note": "same step count as value; e2e within +-1% of value is run-to-run noise, not a gain"},
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "parity": par,
            "variants": variants or None,
            "impl": "b200",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--pairs-per-gpu", type=int, default=64)
    ap.add_argument("--doc-len", type=int, default=4086)
    ap.add_argument("--varlen", action="store_true", help="doc lengths ~U{54..doc_len} instead of fixed")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the forward as a CUDA graph (auto: passages)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--prune-last-layer", action="store_true",
                    help="score with the last layer on the [CLS] rows only (CrossEncoder(prune_last_layer=True))")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU oracle timing (cpu_baseline)")
    ap.add_argument("--ref-budget", type=float, default=120.0, help="seconds of timed pairs in --impl reference")
    ap.add_argument("--no-variants", action="store_true", help="skip the passages / sweep / fp32 variants")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N > 1: process group backend (gloo: test harness, ranks may share a GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
