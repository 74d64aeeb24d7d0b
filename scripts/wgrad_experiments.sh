# conv2 passes at P = 1, 2, 4, 8 (development aid)
cd $GRAFT_REPO_ROOT
for P in 1 2 4 8; do timeout 60 python scripts/pass_bench.py --reps 10 --P $P 2>&1 | tail -1; done
