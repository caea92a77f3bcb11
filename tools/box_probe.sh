# Which kind of GPU box is this (for the host-side D stream)?  Host facts, NT-store bandwidth,
# and the C5 e2e with two ring geometries.  Usage: bash tools/box_probe.sh
lscpu | grep -E "Model name|^CPU\(s\)|L3|NUMA node\(s\)|Thread|Socket" | sed 's/  */ /g'
free -g | head -2
g++ -O2 -mavx512f tools/host_ntbw.cpp -o /tmp/host_ntbw -lpthread && timeout 120 /tmp/host_ntbw | grep -E "T=(1|4|15) " | awk 'NR%2==0'
python tools/d2h_probe.py
for c in 10:2048 16:512; do
  s=${c%%:*}; k=${c##*:}
  PH0B_RING_SLOTS=$s PH0B_RING_CHUNKS=$k timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dropin --e2e-steps 5 > gpurun_out/probe.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/probe.json'));print('ring $c e2e', round(j['e2e']['ms_per_step'],1), 'device', round(j['ms_per_step'],2))"
done
