import sys, math
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np
import oracle
from paper_1709_03187_b200 import make_config_instance
inst = make_config_instance("C5")
xs, ys = inst.xs, inst.ys
n = len(xs)
w = xs.max() - xs.min(); h = ys.max() - ys.min()
cs = math.sqrt(w * h * 2.0 / n)
while True:
    gw = int(w / cs) + 1; gh = int(h / cs) + 1
    L = 3
    while (1 << L) < max(gw, gh): L += 1
    if gw * gh <= 4 * n + 16 and (1 << (2 * L)) <= 16 * n + 4096: break
    cs *= 1.25
cx = ((xs - xs.min()) / cs).astype(np.uint64); cy = ((ys - ys.min()) / cs).astype(np.uint64)
def spread(v):
    v = v & np.uint64(0xffff)
    v = (v | (v << np.uint64(8))) & np.uint64(0x00ff00ff)
    v = (v | (v << np.uint64(4))) & np.uint64(0x0f0f0f0f)
    v = (v | (v << np.uint64(2))) & np.uint64(0x33333333)
    v = (v | (v << np.uint64(1))) & np.uint64(0x55555555)
    return v
key = spread(cx) | (spread(cy) << np.uint64(1))
order = np.lexsort((np.arange(n), key))
int_of = np.empty(n, np.int64); int_of[order] = np.arange(n)
ref = oracle.O2(xs, ys, m=4, k=16, seed=1)
ref.iterate()   # seeding: full constructions
t, l = ref.tours()
ref.iterate(); ref.iterate()
t2, l2 = ref.tours()
for name, tours in (("seeding", t), ("iter3", t2)):
    for a in range(2):
        tour = int_of[tours[a]]
        d = np.abs(np.diff(tour))
        print(name, "ant", a, "median |delta id|", np.median(d), "p75", np.percentile(d, 75), "p90", np.percentile(d, 90))
        for P in (64, 128, 256, 512):
            base = -10**9; hits = 0; restages = 0
            for c in tour:
                if base <= c < base + P: hits += 1
                else:
                    restages += 1
                    base = max(0, min(n - P, c - P // 2))
            print("   P", P, "hit rate", round(hits / n, 3), "restages per 1000 decisions", round(1000 * restages / n, 1))

print("LRU multi-slot policy (restage the least recently used slot on a miss, centred on the missed city; the restage lands `lat` decisions later)")
tour = int_of[t2[0]]
for P, K in ((32, 2), (32, 4), (64, 1), (64, 2), (64, 3), (64, 4), (128, 1), (128, 2)):
    for lat in (0, 4):
        bases = [-10**9] * K; ready = [0] * K; last = [0] * K
        hits = 0
        for i, c in enumerate(tour):
            hit = False
            for s in range(K):
                if bases[s] <= c < bases[s] + P and ready[s] <= i:
                    hit = True; last[s] = i; break
            if hit: hits += 1
            else:
                covered = any(bases[s] <= c < bases[s] + P for s in range(K))  # in flight already
                if not covered:
                    s = min(range(K), key=lambda q: last[q])
                    bases[s] = max(0, min(n - P, c - P // 2)); ready[s] = i + lat; last[s] = i
        print("  P", P, "slots", K, "KB", P * K * 128 // 1024, "lat", lat, "hit rate", round(hits / n, 3))
