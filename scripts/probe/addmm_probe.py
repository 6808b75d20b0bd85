import torch
a = torch.randn(131168, 1536, device="cuda").half(); b = torch.randn(768, 1536, device="cuda").half()
c = torch.mm(a, b.t(), out_dtype=torch.float32)
ref = c.clone()
h0 = a[:, :768]; g0 = b[:, 768:]
try:
    r = torch.addmm(c, h0, g0.t(), beta=0.5, alpha=0.5, out_dtype=torch.float32, out=c)
    print("out= ok, same storage:", r.data_ptr() == c.data_ptr())
    exp = 0.5 * ref + 0.5 * torch.mm(h0, g0.t(), out_dtype=torch.float32)
    print("max diff", (c - exp).abs().max().item())
except Exception as e:
    print("out= failed:", e)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    torch.addmm(c, h0, g0.t(), beta=0.5, alpha=0.5, out_dtype=torch.float32, out=c); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=5, max_name_column_width=60))
bias = torch.randn(768, device="cuda")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    torch.addmm(bias, a, b.t(), out_dtype=torch.float32); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=5, max_name_column_width=60))
