#!/bin/bash
# Round-end evidence on one B200: smoke, the GPU test suite, the bench (both arms), the ncu
# launch list of the bench command, and one ncu --set full capture of the dominant kernel.
# Usage: tools/final_gpu_run.sh <tag>
tag=${1:-final}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_$tag.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc $?" >> gpurun_out/bench_$tag.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
# the launch list of the bench command (cold-cache, serialised: compare shares, not absolutes)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$tag.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
      > gpurun_out/ncu_launches_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_onesweep_p -s 12 -c 1 \
    -o gpurun_out/onesweep_$tag python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-dropin \
    > gpurun_out/ncu_full_$tag.log 2>&1
tail -2 gpurun_out/smoke_$tag.log gpurun_out/pytest_$tag.log; head -c 300 gpurun_out/bench_$tag.json
