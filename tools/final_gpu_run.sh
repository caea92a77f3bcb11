# Round-end evidence on one B200: GPU tests, smoke, bench (both arms), ncu launch list of the
# bench command, ncu --set full of the C5 sort/unique kernels.  Outputs under gpurun_out/.
mkdir -p gpurun_out
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 \
  --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"k2_onesweep_p|k3_unique_p|k1_distance" -c 6 -o gpurun_out/c5_full \
  python tools/run_once.py --config C5 --reps 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
