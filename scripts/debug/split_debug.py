"""Debug the split path on one small case: compare KA's x1 list and the final y with numpy."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import cats_synth
import paper_2404_08763_b200 as cats

def al(v): return (v + 255) // 256 * 256
d, m, b = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dt = torch.float32 if sys.argv[4] == "f32" else torch.bfloat16
es = 4 if dt == torch.float32 else 2
Wg, Wu, Wd = cats_synth.mlp_weights(d, m, dt, layer=0)
x = cats_synth.tokens(b, d, dt, seed=1)
plan = cats.MlpPlan(d, m, max_batch=b, dtype=dt)
ws = plan.workspace()
t = 0.05
y = cats.cats_mlp_decode(plan, x.cuda(), Wg.cuda(), Wu.cuda(), Wd.cuda(), t, ws=ws).cpu().double().numpy()
torch.cuda.synchronize()
off = 0; o = {}
o["sched"] = off; off = al(off + 64)
o["idx"] = off; off = al(off + m * 4)
o["tm"] = off; off = al(off + m)
o["vals"] = off; off = al(off + m * b * 4)
o["cnt"] = off; off = al(off + (m + 1) // 2 * 4)
o["ypart"] = off; off = al(off + b * d * 8)
o["xs"] = off; off = al(off + b * d * es)
o["ys"] = off; off = al(off + b * d * 4)
o["x1"] = off
w = ws.cpu().numpy()
NR = plan.info["rows_per_tile"]
ntiles = (m + NR - 1) // NR
cnt = w[o["cnt"]:o["cnt"] + ntiles * 4].view(np.int32)
idxa = w[o["idx"]:o["idx"] + m * 4].view(np.int32)
x1 = w[o["x1"]:o["x1"] + ntiles * NR * b * 4].view(np.float32).reshape(-1, b)
sched = w[:64].view(np.uint32)
print("sched", sched[:4], "U", cnt.sum(), "NR", NR)
X = x.float().double().numpy(); G = Wg.float().double().numpy(); Uu = Wu.float().double().numpy(); D = Wd.float().double().numpy()
u = X @ G.T; v = u / (1 + np.exp(-u)); keep = np.abs(v) >= t
up = X @ Uu.T
x1ref = up * v * keep
bad = 0
for tile in range(ntiles):
    for k in range(cnt[tile]):
        pos = tile * NR + k
        j = idxa[pos]
        if not np.allclose(x1[pos], x1ref[:, j], rtol=1e-3, atol=1e-5):
            bad += 1
            if bad < 5: print("x1 mismatch pos", pos, "j", j, x1[pos], x1ref[:, j])
print("x1 mismatches", bad)
yref = x1ref @ D
err = np.linalg.norm(y - yref) / np.linalg.norm(yref)
print("y rel err", err)
print("y[0,:8]", y[0, :8]); print("ref[0,:8]", yref[0, :8])
