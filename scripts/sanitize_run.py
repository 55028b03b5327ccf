"""Small-shape workload touching every kernel family once, for checking runs: compute-sanitizer where the
pool allows it (closed on this pool), and the debug library's device-side bounds checks:

    python -m paper_2404_08763_b200.build --debug && python scripts/sanitize_run.py --debug
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

if "--debug" in sys.argv:  # load libcats_debug.so (CATS_DCHECK compiled in) instead of libcats.so
    from paper_2404_08763_b200 import _lib
    _lib.LIB_PATH = _lib.LIB_PATH.replace("libcats.so", "libcats_debug.so")

import cats_synth
import paper_2404_08763_b200 as cats
from paper_2404_08763_b200 import tp

dev = "cuda"
d, m = 512, 1000
Wg, Wu, Wd = (w.to(dev) for w in cats_synth.mlp_weights(d, m, torch.bfloat16))
for opts in ({}, {"path": cats.CATS_PATH_FUSED}, {"path": cats.CATS_PATH_FUSED, "lazy_tail": 0, "eager": 1}, {"compaction": cats.CATS_COMPACT_PREDICATED},
             {"compaction": cats.CATS_COMPACT_ATOMIC}, {"path": cats.CATS_PATH_SPLIT}):
    plan = cats.MlpPlan(d, m, max_batch=8, **opts)
    ws = plan.workspace()
    for b in (1, 2, 4):
        x = cats_synth.tokens(b, d, torch.bfloat16, seed=b).to(dev)
        for _ in range(2):
            cats.cats_mlp_decode(plan, x, Wg, Wu, Wd, 0.05, ws=ws)
        cats.cats_mlp_dense(plan, x, Wg, Wu, Wd, ws=ws)
        cats.cats_mlp_last_active(plan, ws, b)
    print("decode", opts, "ok", flush=True)
# wide rows (d = 5120: KA + KB at b = 1, MMA KB with 5 tiles per warp at b = 4)
d2, m2 = 5120, 1728
W2 = [w.to(dev) for w in cats_synth.mlp_weights(d2, m2, torch.bfloat16)]
p2 = cats.MlpPlan(d2, m2, max_batch=4)
ws2 = p2.workspace()
for b in (1, 4):
    cats.cats_mlp_decode(p2, cats_synth.tokens(b, d2, torch.bfloat16).to(dev), *W2, 0.05, ws=ws2)
acts = cats.cats_mlp_gate_act(p2, cats_synth.tokens(4, d2, torch.bfloat16).to(dev), W2[0], ws=ws2)
# KA in column parts (d = 5120, b >= 6: 8-row tiles, 1024-column stages), ragged m
p3 = cats.MlpPlan(d2, 1003, max_batch=8)
W3 = [w.to(dev) for w in cats_synth.mlp_weights(d2, 1003, torch.bfloat16)]
ws3 = p3.workspace()
for b in (6, 8):
    cats.cats_mlp_decode(p3, cats_synth.tokens(b, d2, torch.bfloat16).to(dev), *W3, 0.05, ws=ws3)
    cats.cats_mlp_last_active(p3, ws3, b)
# bound host call (graph: x staging kernel + decode kernels), K12 and the split path
hp = cats.MlpPlan(d, m, max_batch=2)
hws = hp.workspace()
for b in (1, 2):
    xh = cats_synth.tokens(b, d, torch.bfloat16).pin_memory()
    call = cats.BoundDecodeHost(hp, xh, Wg, Wu, Wd, 0.05, ws=hws)
    for _ in range(3):
        call()
print("wide ok", flush=True)
# App. B input-sparse projection
xp = cats.XsparsePlan(512, 768, max_batch=8)
Wx = cats_synth.attn_weights(512, 768).to(dev)
for b in (1, 3, 8):
    cats.cats_xsparse_gemv(xp, cats_synth.tokens(b, 512, torch.bfloat16).to(dev), Wx, 0.5, ws=xp.workspace())
print("xsparse ok", flush=True)
# calibration: small (register-load kernel), large enough for the TMA ring kernel, fp32 multi-pass
for n, dt in ((100_003, torch.bfloat16), (3_000_000, torch.bfloat16), (1_500_001, torch.float32)):
    a = cats_synth.calib_acts(n, dt, device=dev)
    cats.cats_calibrate_threshold(a, 0.7)
print("calib ok", flush=True)
# fused TP reduction, 4 emulated ranks, a few epochs
em = tp.EmulatedTpComms(4, 2048)
for _ in range(3):
    em.allreduce([torch.randn(2048, device=dev) for _ in range(4)])
torch.cuda.synchronize()
print("tp ok", flush=True)
print("library:", cats.library_path(), flush=True)
