#!/bin/bash
# full validation of HEAD: smoke, every -m gpu test (incl. slow), the bench line
cd "${GRAFT_REPO_ROOT:-.}"
tag=${1:-full}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 3000 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_tests.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${tag}_bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${tag}_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/${tag}_ref.log
