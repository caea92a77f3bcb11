# e2e A/B of the D2H ring geometry: "slots:chunks" pairs in $CFGS (two runs each)
for rep in 1 2; do for c in $CFGS; do
  s=${c%%:*}; k=${c##*:}
  PH0B_RING_SLOTS=$s PH0B_RING_CHUNKS=$k timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dropin --e2e-steps 5 > gpurun_out/ring.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/ring.json'));print('slots=$s chunks=$k e2e', round(j['e2e']['ms_per_step'],1), j['e2e']['check'])"
done; done
