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
            f"s={s}), w=4 asymmetric, packed varlen batch (BASELINE configs[2])")


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

def cpu_oracle_layer_times(cfg, doc_len, reps, budget_s=None):
    from oracle import sparsecross_oracle as O

    ocfg = dict(cfg)
    wt = O.init_weights(ocfg, 0, np.float32)
    ids, spans = O.gen_random_ids(0, QUERY_LEN, doc_len, 1, cfg["vocab_size"])
    x = O.embed(ids, wt, np.float32)
    pattern = O.resolve_pattern(ocfg, spans)
    times = []
    t_start = time.perf_counter()
    for r in range(reps):
        t0 = time.perf_counter()
        O.layer_forward(x, spans, pattern, wt, r % cfg["layers"], ocfg)
        times.append(time.perf_counter() - t0)
        if budget_s and time.perf_counter() - t_start > budget_s and len(times) >= 3:
            break
    return times


def cpu_threads():
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
        if os.environ.get(v, "").isdigit():
            return int(os.environ[v])
    return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, doc_len, s = workload(args)
    times = cpu_oracle_layer_times(cfg, doc_len, args.warmup + args.steps)
    timed = times[args.warmup:] or times
    t_layer = statistics.median(timed)
    value = 1.0 / (cfg["layers"] * t_layer)
    sample = (f"1 pair at s={s} (q{QUERY_LEN}+d{doc_len}), 1 of {cfg['layers']} identical encoder layers per step, "
              f"f32 numpy oracle port of R/encoder.py:306-371; pairs/s = 1/(layers * median layer time)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": args.gpus,
        "steps": len(timed), "warmup": args.warmup, "ms_per_step": t_layer * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generator ids, seed 0)",
        "config": {"workload": workload_name(doc_len, s), "seq_len": s,
                   "doc_len": doc_len, "query_len": QUERY_LEN, "window": 4, "pattern": "sparse"},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cpu_threads(), "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


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
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
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
        if world > 1:
            dist.all_gather_into_tensor(gathered, scores)
            return gathered
        return scores

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
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
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
    e2e_steps = max(3, args.steps // 2)
    for _ in range(e2e_steps):
        e2e_step()
    f1.record(stream)
    barrier()
    te = torch.tensor([f0.elapsed_time(f1)], device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = n * world * e2e_steps / (float(te.item()) / 1e3)

    # ---- variant: last layer on the [CLS] rows only (opt-in serving mode) ----
    variants = None
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
        tv = torch.tensor([v0.elapsed_time(v1)], device=dev)
        if world > 1:
            dist.all_reduce(tv, op=dist.ReduceOp.MAX)
        model.prune_last_layer = False
        variants = {"prune_last_layer": {
            "value": n * world * vsteps / (float(tv.item()) / 1e3), "unit": "pairs/s", "steps": vsteps,
            "note": "CrossEncoder(prune_last_layer=True): last layer past K/V on the [CLS] rows only (the score "
                    "reads x[:,0], R/encoder.py:506); same scores, not the headline"}}

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
        times = cpu_oracle_layer_times(cfg, doc_len, reps=50, budget_s=args.cpu_budget)
        tl = statistics.median(times)
        cpu = {"value": 1.0 / (cfg["layers"] * tl), "unit": "pairs/s", "cores": cpu_threads(), "kind": "port",
               "sample": f"1 pair at s={s}, {len(times)} x 1-of-{cfg['layers']} encoder layers (f32 numpy oracle port, "
                         f"R/encoder.py:306-371), median {tl * 1e3:.1f} ms/layer; pairs/s = 1/(layers * layer time)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: reference-generator token ids (default_rng((seed,q,i))), random-init ELECTRA-base weights",
            "config": {"workload": workload_name(doc_len, s), "cuda_graph": use_graph, "prune_last_layer": bool(args.prune_last_layer),
                       "pairs_per_gpu": n, "global_batch": n * world, "seq_len": s, "doc_len": doc_len,
                       "query_len": QUERY_LEN, "varlen": bool(args.varlen), "pattern": "sparse", "window": 4,
                       "layers": 12, "hidden": 768, "heads": 12, "ff": 3072, "parallelism": f"dp{world}",
                       "l2": f"inputs larger than L2 (qkv activations {layout.total_tokens * 2304 * 2 / 1e9:.2f} GB per layer)"},
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
                    "d2h_bytes_per_step": int(host_scores.numel() * 4)},
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "variants": variants,
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
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU oracle timing")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
