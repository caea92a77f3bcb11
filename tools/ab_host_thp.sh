# (Experiment record: the PH0B_HOST_THP code path this script toggles was measured and reverted —
#  see commit 445edd6 and DESIGN.md "Tried".)
# process-to-process spread of the host-path e2e with pinned buffers from cudaHostAlloc (0) or
# THP + cudaHostRegister (1); ring geometry fixed at 10 x 8 MiB so slow processes show
for rep in 1 2 3 4 5 6; do for v in 0 1; do
  PH0B_HOST_THP=$v PH0B_RING_TUNE=0 timeout 600 python tools/e2e_once.py --reps 4 2>/dev/null | tail -3 | awk -v v=$v '{print "thp=" v, $0}' | cut -c1-40
done; done
