import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, cats_synth, paper_2404_08763_b200 as cats
d, m, b = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
heavy = len(sys.argv) > 4
Wg, Wu, Wd = (w.cuda() for w in cats_synth.mlp_weights(d, m, torch.bfloat16, layer=7, heavy=heavy))
x = cats_synth.tokens(b, d, torch.bfloat16, seed=8, heavy=heavy).cuda()
plan = cats.MlpPlan(d, m, max_batch=b)
ws = plan.workspace()
for i in range(3):
    y = cats.cats_mlp_decode(plan, x, Wg, Wu, Wd, 0.1, ws=ws)
    torch.cuda.synchronize()
print("ok", float(y.abs().sum()))
X = x.double(); G = Wg.double(); Uu = Wu.double(); D = Wd.double()
u = X @ G.T; v = u / (1 + torch.exp(-u)); keep = v.abs() >= 0.1
yref = ((v * keep) * (X @ Uu.T)) @ D
err = ((y.double() - yref).norm(dim=1) / yref.norm(dim=1)).cpu().numpy()
print("per-token rel err", err.round(5))
q = (y.double() - yref).abs().cpu()
for part in range(4):
    cols = slice(part * d // 4, (part + 1) * d // 4)
    print("part", part, "max abs err", float(q[:, cols].max()), "zero frac", float((y[:, cols] == 0).float().mean()))
