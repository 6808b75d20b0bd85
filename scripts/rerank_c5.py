"""C5 driver: synthetic TREC-DL-style re-ranking (queries x top-k documents at 4096 tokens)
over 1..8 GPUs, one process per GPU (BASELINE.json configs[4]).

  python scripts/rerank_c5.py --queries 20                      # 1 GPU
  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 scripts/rerank_c5.py --queries 1000

Each rank scores a contiguous block of queries (ELECTRA-base sparse w=4, bf16,
random-init weights); scores are gathered with one NCCL all-gather; rank 0
ranks them with the reference tie-break (-score, candidate position), writes
the TREC run file and prints one JSON line.  Throughput counts the whole job
(host packing + GPU scoring + gather + ranking): pairs / wall-clock seconds of
the slowest rank, timed after a warm-up query.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17649_b200 as P  # noqa: E402
from paper_2312_17649_b200.rerank import rerank_distributed, synthetic_queries, write_run  # noqa: E402

ELECTRA = dict(layers=12, embed_dim=768, heads=12, ff_dim=3072, vocab_size=30522, pattern="sparse", window=4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--queries", type=int, default=20)
    ap.add_argument("--docs", type=int, default=100)
    ap.add_argument("--doc-len", type=int, default=4086)
    ap.add_argument("--top-k", type=int, default=100)
    ap.add_argument("--prune-last-layer", action="store_true")
    ap.add_argument("--run-file", default=None)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    s = 10 + args.doc_len + 3
    cfg = P.EncoderConfig(**ELECTRA, max_positions=max(s, 512), precision="bf16")
    model = P.CrossEncoder(cfg, seed=0, device=dev, prune_last_layer=args.prune_last_layer)
    # every rank generates only its own shard of the synthetic candidates
    from paper_2312_17649_b200.rerank import shard_range
    lo, hi = shard_range(args.queries, world, rank)
    mine = synthetic_queries(hi - lo, args.docs, args.doc_len, cfg.vocab_size, qid_offset=lo)
    placeholder = [(f"q{q}", None, [(f"d{q}_{i}", None) for i in range(args.docs)]) for q in range(args.queries)]
    queries = placeholder[:lo] + mine + placeholder[hi:]
    # warm-up (one query on every rank, not counted)
    warm = synthetic_queries(1, min(args.docs, 8), args.doc_len, cfg.vocab_size, qid_offset=10 ** 6)
    rerank_distributed(model, warm, top_k=8)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    entries = rerank_distributed(model, queries, top_k=args.top_k, rank=rank, world=world)
    torch.cuda.synchronize()
    t = torch.tensor([time.perf_counter() - t0], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    secs = float(t.item())
    if rank == 0:
        if args.run_file:
            write_run(entries, args.run_file)
        pairs = args.queries * args.docs
        print(json.dumps({
            "metric": "re-ranked query-doc pairs/sec (whole job, wall clock)", "value": pairs / secs,
            "unit": "pairs/s", "n_gpus": world, "queries": args.queries, "docs_per_query": args.docs,
            "seq_len": s, "seconds": secs, "run_entries": len(entries),
            "config": "ELECTRA-base sparse w=4 bf16, synthetic ids default_rng((0, q, i)), random-init weights "
                      "(BASELINE configs[4])", "prune_last_layer": bool(args.prune_last_layer)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
