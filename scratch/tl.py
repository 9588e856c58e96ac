import sys, re
rows=[tuple(int(x) for x in re.findall(r'-?\d+', l)) for l in open(sys.argv[1]) if l.startswith('TL')]
t0=min(r[4] for r in rows)
starts=sorted((r[4]-t0)/1e3 for r in rows); ends=sorted((r[5]-t0)/1e3 for r in rows)
print("ctas", len(rows), "start us: min %.1f med %.1f max %.1f" % (starts[0], starts[len(starts)//2], starts[-1]), " end us: min %.1f med %.1f max %.1f" % (ends[0], ends[len(ends)//2], ends[-1]))
sms=[r[3] for r in rows]; from collections import Counter; c=Counter(sms); print("distinct SMs", len(c), "max ctas/SM", max(c.values()))
late=[r for r in rows if (r[4]-t0)/1e3 > 50]; print("late ctas", len(late), "items", sorted(set(r[1] for r in late))[:20])
