# HBM access-pattern probe: in-place read+write over 12-position chunks (no arithmetic)
cd $GRAFT_REPO_ROOT
B=scripts/dev/pattern_bw
for p in 0,1,2,3,4,5,6,7,8,9,10,11 0,1,2,3,4,5,6,7,12,19,21,28 0,1,2,8,9,10,11,12,13,14,15,16 0,1,2,17,18,19,20,21,22,23,24,25 0,1,2,3,4,8,9,17,26,27,28,29 0,1,2,5,6,7,10,11,12,13,14,18 0,1,2,9,13,14,18,19,20,21,28,29 0,1,2,3,4,5,6,9,12,24,25,26 0,1,2,3,4,5,6,7,8,9,10,29; do
  timeout 120 $B 30 $p
done > gpurun_out/pat_bw.jsonl 2>&1
