# e2e A/B of the host path's key-range bucket schedule (PH0B_BUCKETS, cumulative /256)
S0="16,17,19,23,31,47,63,79,95,111,127,143,159,175,191,207,223,239"
S1="32,33,35,39,47,63,79,95,111,127,143,159,175,191,207,223,239"
S2="24,25,27,31,39,55,71,87,103,119,135,151,167,183,199,215,231,247"
S3="32,36,44,60,76,92,108,124,140,156,172,188,204,220,236"
for rep in 1 2; do for i in 0 1 2 3; do
  eval "b=\$S$i"
  PH0B_BUCKETS=$b timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dropin --e2e-steps 5 > gpurun_out/bk.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/bk.json'));print('schedule S$i e2e', round(j['e2e']['ms_per_step'],1), j['e2e']['check']['scale_equal_device_path'])"
done; done
