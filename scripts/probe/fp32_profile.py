"""Kernel time breakdown (torch.profiler) of one fp32 f16x3 step at 32 x s=4099."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_2312_17649_b200 as P
mode = sys.argv[1] if len(sys.argv) > 1 else "f16x3"
cfg = dict(bench.ELECTRA, max_positions=4099)
batch = bench.make_batch(P, cfg, 4086, 32, 0)
model = P.CrossEncoder(P.EncoderConfig(**cfg, precision="f32"), seed=0, device="cuda", fp32_gemm=mode)
layout = model.make_layout(batch)
ids = torch.from_numpy(batch.ids).cuda()
fn = lambda: model.scores_from_hidden(model.encode_packed(ids, layout), layout)
for _ in range(2): fn()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    fn(); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=90))
