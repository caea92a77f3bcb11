# drop-in (ph0b_h0_barcode) e2e with the library's result buffer pinned vs anonymous mapping
for rep in 1 2; do for v in 1 0; do
  PH0B_PINNED_RESULTS=$v PH0B_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pr.json 2> gpurun_out/pr.err
  python -c "import json;j=json.load(open('gpurun_out/pr.json'));print('pinned_results=$v e2e', round(j['e2e']['ms_per_step'],1), 'dropin', round(j['e2e_dropin']['ms_per_step'],1), j['e2e_dropin']['check'])"
  grep "D2H ring" gpurun_out/pr.err | tail -1
done; done
