"""A/B timing of K1+K2 under different environment settings (same library),
interleaved rounds.  usage: python scratch/ab_env.py B T S 'ENV=..' 'ENV=..' ..."""
import sys, os, subprocess, json
B, T, S = sys.argv[1:4]
variants = sys.argv[4:]
code = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ab.py")).read()
code = code[code.index("code = r'''") + 11: code.index("''' % (B, T, S)")] % (B, T, S)
res = {v: [] for v in variants}
for rnd in range(3):
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            if "=" in kv:
                k, val = kv.split("=", 1)
                env[k] = val
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
        try:
            res[v].append(json.loads(r.stdout.strip().splitlines()[-1]))
        except Exception:
            print(v, r.stderr[-800:])
for v in variants:
    rs = res[v]
    if not rs:
        continue
    print(f"{v:40s} fwd min {min(x['fwd_min'] for x in rs):7.1f}  med {sorted(x['fwd_med'] for x in rs)[len(rs)//2]:7.1f}  bt {rs[0]['bt_med']:5.1f}  clk {[x['clk'] for x in rs]}")
