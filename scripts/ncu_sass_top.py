"""Top SASS instructions by warp-stall samples from an `ncu --page source --csv --print-source sass` export."""
import csv, sys

def main(path, n=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    idx = {k: i for i, k in enumerate(hdr)}
    data = rows[2:]
    tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
    print(f"total samples {tot}, instructions {len(data)}")
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    top = sorted(data, key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))[:n]
    for r in top:
        samp = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        reasons = sorted(((int(r[idx[c]] or 0), c[6:]) for c in cols), reverse=True)[:3]
        print(f"{samp / tot * 100:5.1f}% {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:60]:60s} "
              + " ".join(f"{c}:{v}" for v, c in reasons if v))
    # local memory (spill) traffic
    loc = [r for r in data if "LDL" in r[idx["Source"]] or "STL" in r[idx["Source"]]]
    print("local-memory instructions:", len(loc), "samples", sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in loc),
          "executed", sum(int(r[idx["Instructions Executed"]] or 0) for r in loc))

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
