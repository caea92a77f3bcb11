# usage: bash tools/ring_sweep.sh "G,R,S,NS" ...   (D2H ring: chunks per piece, slots,
# copy streams, decode tasks per piece)
mkdir -p gpurun_out; : > gpurun_out/sweep.log
for cfg in "$@"; do
  IFS=, read -r G R S NS <<< "$cfg"
  echo "== G=$G R=$R S=$S NS=$NS" >> gpurun_out/sweep.log
  PH0B_RING_CHUNKS=$G PH0B_RING_SLOTS=$R PH0B_RING_STREAMS=$S PH0B_RING_SUBTASKS=$NS PH0B_TRACE=1 \
    timeout 120 python tools/e2e_once.py --reps 3 2>&1 | grep -E "^rep|pieces" | sed 's/stages.*//' >> gpurun_out/sweep.log
done
