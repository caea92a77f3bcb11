# A/B of kernel variants selected by an env knob: VAR=<env name> VALS="a b c" tools/ab_exp.sh
mkdir -p gpurun_out; : > gpurun_out/ab_exp.txt
for rep in 1 2; do for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dropin --e2e-steps 1 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "import json;j=json.load(open('gpurun_out/ab_$v.json'));print('$VAR=$v', round(j['ms_per_step'],3), j['roofline']['avg_launch_ms'], j['stage_ms']['unique_ms'], j['e2e']['check'])" >> gpurun_out/ab_exp.txt 2>&1
done; done
cat gpurun_out/ab_exp.txt
