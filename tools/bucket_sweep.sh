# usage: bash tools/bucket_sweep.sh "c1,c2,..." ...  (bucket schedules of the host path)
mkdir -p gpurun_out; : > gpurun_out/bsweep.log
for cfg in "$@"; do
  echo "== $cfg" >> gpurun_out/bsweep.log
  PH0B_BUCKETS=$cfg timeout 120 python tools/e2e_once.py --reps 4 2>&1 | grep -E "^rep" | sed 's/stages.*//' >> gpurun_out/bsweep.log
done
