"""Data-parallel fine-tuning across GPUs (one process per GPU, NCCL all-reduce of the flat
gradient buffer), ELECTRA-base dims, synthetic packed pairs.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 scripts/train_dp.py

Each rank trains on its own batches; the weights stay identical across ranks (checked at the end
with an all-gathered checksum).  Prints one JSON line on rank 0 (whole-job tokens/s, max over
ranks of the device-timed steps).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17649_b200 as P  # noqa: E402
from paper_2312_17649_b200 import training as TR  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--doc-len", type=int, default=4086)
    ap.add_argument("--pairs", type=int, default=4)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1 or "RANK" in os.environ:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    s = 10 + a.doc_len + 3
    cfg = P.EncoderConfig(layers=12, embed_dim=768, heads=12, ff_dim=3072, max_positions=s, vocab_size=30522,
                          pattern="sparse", window=4, precision="bf16")
    model = TR.TrainableCrossEncoder(cfg, seed=0)  # same init on every rank
    opt = TR.AdamW(1e-5)
    part = P.SubsequencePartition((0, 1), (1, 12), (12, s))
    rng = np.random.default_rng(1000 + rank)

    def batch_ids():
        ids = rng.integers(3, cfg.vocab_size, size=(2 * a.pairs, s)).astype(np.int32)
        ids[:, 0], ids[:, 11], ids[:, -1] = 1, 2, 2
        return ids

    batch = P.PackedBatch.from_ids(batch_ids(), part)
    step = TR.GraphedTrainStep(model, opt, batch, process_group=None)
    gaps = rng.standard_normal(a.pairs)
    for _ in range(a.warmup):
        step(batch_ids().reshape(-1), gaps)
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        loss = step(batch_ids().reshape(-1), gaps)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / a.steps], device="cuda")
    chk = model.weights.flat.double().sum().reshape(1)
    if dist.is_initialized():
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        allc = [torch.zeros_like(chk) for _ in range(world)]
        dist.all_gather(allc, chk)
        assert all(torch.equal(c, allc[0]) for c in allc), "weights diverged across ranks"
    if rank == 0:
        tokens = batch.total_tokens * world
        print(json.dumps({"metric": "dp_finetune_step", "n_gpus": world, "ms_per_step": float(ms),
                          "tokens_per_s": tokens / float(ms) * 1e3, "pairs_per_s": 2 * a.pairs * world / float(ms) * 1e3,
                          "loss": float(loss), "scaling": "weak"}))
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
