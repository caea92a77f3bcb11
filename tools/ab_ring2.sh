# bad-box knobs around the 16 x 512 ring: copy streams and decode tasks per piece
export PH0B_RING_SLOTS=16 PH0B_RING_CHUNKS=512
for rep in 1 2; do for c in 2:32 3:32 1:32 2:16 2:64; do
  st=${c%%:*}; sub=${c##*:}
  PH0B_RING_STREAMS=$st PH0B_RING_SUBTASKS=$sub timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dropin --e2e-steps 5 > gpurun_out/r2.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/r2.json'));print('streams=$st subtasks=$sub e2e', round(j['e2e']['ms_per_step'],1))"
done; done
