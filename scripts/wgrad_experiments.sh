# conv2 passes at P = 1, 2, 4, 8: stream tail on / off (development aid)
cd $GRAFT_REPO_ROOT
for P in 1 2 4 8; do for t in 1 0; do echo -n "stream=$t "; CP_TC_STREAM_TAIL=$t timeout 60 python scripts/pass_bench.py --reps 10 --P $P 2>&1 | tail -1; done; done
