import sys, re, numpy as np
d={}
for l in open(sys.argv[1]):
    m=re.match(r'BT (\d+) (\d+) (\d+) (\d+)',l)
    if m: d[(int(m[1]),int(m[2]))]=(int(m[3]),int(m[4]))
if not d: print("no BT lines"); sys.exit()
t=np.array([v[0] for v in d.values()])/1e3; ns=np.array([v[1] for v in d.values()])
blocks=sorted({k[0] for k in d})
bt=np.array([max(d[(b,w)][0] for (bb,w) in d if bb==b) for b in blocks])/1e3
print(f"warps {len(t)}: mean {t.mean():.1f} us, max {t.max():.1f}, min {t.min():.1f}, p95 {np.percentile(t,95):.1f}; searches/warp mean {ns.mean():.0f} max {ns.max()} min {ns.min()}")
print(f"blocks {len(bt)}: mean-of-block-max {bt.mean():.1f} us, max {bt.max():.1f}, min {bt.min():.1f}")
bm=np.array([np.mean([d[(b,w)][0] for (bb,w) in d if bb==b]) for b in blocks])/1e3
print(f"per-block mean warp time: mean {bm.mean():.1f}, min {bm.min():.1f}, max {bm.max():.1f}")
