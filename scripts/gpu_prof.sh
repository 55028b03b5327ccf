#!/bin/bash
# ncu launch list + full capture of K1/K2/K3 at the bench shape. Logs to gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
CMD="python scripts/prof_decode.py --steps 8 --dense ${PROF_ARGS}"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/prof_plain.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k12_" -s 10 -c 2 \
   -o gpurun_out/${TAG}_prof -f $CMD > gpurun_out/ncu_full.log 2>&1
# read-bandwidth ceilings with torch (context): sum (read-only) and copy of 4 GiB
timeout 120 python - > gpurun_out/membw.log 2>&1 <<'PY'
import torch
x = torch.empty(2*1024**3, dtype=torch.bfloat16, device="cuda").normal_()
y = torch.empty_like(x)
for name, fn, nbytes in [("sum", lambda: x.sum(dtype=torch.float32), x.numel()*2), ("copy", lambda: y.copy_(x), x.numel()*4)]:
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)/10
    print(name, round(nbytes/ms/1e6, 1), "GB/s")
PY
ls -la gpurun_out/
