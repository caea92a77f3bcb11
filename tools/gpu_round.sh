#!/bin/bash
# One validation pass on the GPU box: smoke, the GPU test suite, the bench (both arms).
# Usage: tools/gpu_round.sh <tag> [pytest-args...]
tag=${1:-run}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest tests -m gpu -x -q ${@} > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_$tag.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc $?" >> gpurun_out/bench_$tag.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
tail -3 gpurun_out/smoke_$tag.log gpurun_out/pytest_$tag.log; cat gpurun_out/bench_$tag.json
