for rep in 1 2; do for t in 15 12 16 20; do
  PH0B_DECODE_THREADS=$t timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dropin --e2e-steps 5 > gpurun_out/dt.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/dt.json'));print('threads=$t e2e', round(j['e2e']['ms_per_step'],1))"
done; done
