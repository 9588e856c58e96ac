"""Summarise tools/ncu_source.sh output: stall-sample shares of K1's fast
stage body and of the per-stage bookkeeping around it (instructions grouped
by execution count), plus the top instructions.
usage: python tools/ncu_source_summary.py gpurun_out/fwd_<tag>_source.csv"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
by = collections.defaultdict(lambda: [0, 0, collections.Counter()])
tot = 0
for r in data:
    try:
        ex = int(r[ix["Instructions Executed"]])
        s = int(r[ix["# Samples"]])
    except (ValueError, KeyError):
        continue
    tot += s
    g = by[ex]
    g[0] += s
    g[1] += 1
    for h in reasons:
        try:
            g[2][h] += int(r[ix[h]])
        except ValueError:
            pass
print("total samples", tot)
for ex, (s, n, c) in sorted(by.items(), key=lambda kv: -kv[1][0])[:8]:
    t = max(1, sum(c.values()))
    print(f"exec {ex:9d}: {n:4d} instrs, {s:5d} samples ({s / tot * 100:.1f}%): " +
          ", ".join(f"{k[6:]} {v / t * 100:.0f}%" for k, v in c.most_common(5)))
