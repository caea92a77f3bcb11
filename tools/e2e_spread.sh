# C5 host-path e2e in N separate processes (default settings): the process-to-process spread
N=${N:-8}
for p in $(seq 1 $N); do
  timeout 600 python tools/e2e_once.py --reps 6 2>/dev/null | tail -4 | awk -v p=$p '{printf "proc %d %s  ", p, $3} END {print ""}'
done
