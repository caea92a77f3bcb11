# e2e A/B of an env knob: VAR=<env name> VALS="a b c" tools/ab_e2e.sh (two runs each)
for rep in 1 2; do for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dropin --e2e-steps 5 > gpurun_out/abe.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/abe.json'));print('$VAR=$v e2e', round(j['e2e']['ms_per_step'],1), round(j['e2e']['d2h_bytes_per_step']/1e9,2), 'GB', j['e2e']['check'])"
done; done
