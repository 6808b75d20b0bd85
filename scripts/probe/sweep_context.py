"""Does the attention sweep depend on what ran before it?  sweep cold -> 10 bf16 encoder steps ->
sweep -> 3 s idle -> sweep, with nvidia-smi clocks sampled during each sweep."""
import json, math, os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench
import paper_2312_17649_b200 as P

hbm, tf, _, _ = bench.peaks()
dev = torch.device("cuda")
wins = (("sparse", 4), ("sparse", 64), ("sparse", 256))


def sweep(tag):
    with bench.ClockSampler(0) as clk:
        res = bench.attention_sweep(P, dev, (hbm, tf), windows=wins)
    print(tag, [(p["window"], p["us_per_seq_layer"], p["frac_of_bound"]) for p in res["points"]], clk.summary(), flush=True)


sweep("cold")
cfg = dict(bench.ELECTRA, max_positions=4099)
model = P.CrossEncoder(P.EncoderConfig(**cfg, precision="bf16"), seed=0, device=dev)
batch = bench.make_batch(P, cfg, 4086, 64, 0)
layout = model.make_layout(batch)
ids = torch.from_numpy(batch.ids).to(dev)
for _ in range(10):
    model.scores_from_hidden(model.encode_packed(ids, layout), layout)
torch.cuda.synchronize()
sweep("after_steps")
time.sleep(3)
sweep("after_idle3s")
del model
torch.cuda.empty_cache()
sweep("after_free")
