"""Kernel-level sweep (C4): packed batch of 4099-token sequences, H=12, d=64, bf16.

Times sc_attn_fwd with CUDA events on the launching stream and reports the
algorithmic-byte roofline (4*s*h*2 bytes per sequence-layer).
"""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17649_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nseq", type=int, default=64)
    ap.add_argument("--doc", type=int, default=4086)
    ap.add_argument("--windows", default="1,4,16,64,256,inf")
    ap.add_argument("--patterns", default="sparse")
    ap.add_argument("--algo", default="auto")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--qds-every", type=int, default=30, help="QDS global-token spacing (pattern qds)")
    args = ap.parse_args()
    H, d, m = 12, 64, 10
    s = m + args.doc + 3
    T = s * args.nseq
    lay = P.PackedLayout.from_lengths([s] * args.nseq, [m + 1] * args.nseq)
    lay_qds = None
    g = torch.Generator(device="cuda").manual_seed(0)
    qkv = torch.randn((T, 3 * H * d), device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty((T, H * d), device="cuda", dtype=torch.bfloat16)
    peak = 6553.6
    for pname in args.patterns.split(","):
        for ws in args.windows.split(","):
            w = math.inf if ws == "inf" else int(ws)
            pat = P.make_pattern(pname, w)
            L = lay
            if pname == "qds":  # global doc tokens every --qds-every positions (R/encoder.py:180-184)
                if lay_qds is None:
                    lay_qds = P.PackedLayout.from_lengths([s] * args.nseq, [m + 1] * args.nseq,
                                                          qds_every=args.qds_every)
                L = lay_qds
            f = lambda: P.attend_packed(qkv[:, :H * d], qkv[:, H * d:2 * H * d], qkv[:, 2 * H * d:], L, pat, H,
                                        out=out, algo=args.algo, check=False)
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            st = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.iters):
                f()
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.iters
            byts = 4 * T * H * d * 2
            gbs = byts / ms / 1e6
            print(json.dumps({"pattern": pname, "w": ws, "ms": round(ms, 4), "GB/s": round(gbs, 1),
                              "frac_hbm": round(gbs / peak, 3), "us_per_seq_layer": round(ms * 1e3 / args.nseq, 2)}))


if __name__ == "__main__":
    main()
