# decode-thread count A/B with each ring geometry (C5 e2e, two runs each)
for geo in 16:512 10:2048; do for rep in 1 2; do for t in 13 15 16; do
  PH0B_RING_SLOTS=${geo%%:*} PH0B_RING_CHUNKS=${geo##*:} PH0B_DECODE_THREADS=$t timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dropin --e2e-steps 5 > gpurun_out/dt.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/dt.json'));print('ring $geo threads=$t e2e', round(j['e2e']['ms_per_step'],1))"
done; done; done
