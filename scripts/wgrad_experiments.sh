# conv2 passes at P = 1, 2, 4, 8; wgrad tail piece cap (development aid)
cd $GRAFT_REPO_ROOT
for P in 1 2 4 8; do timeout 60 python scripts/pass_bench.py --reps 10 --P $P 2>&1 | tail -1; done
for m in 8 32 148; do CP_TC_TAIL_MAX=$m timeout 60 python scripts/pass_bench.py --reps 10 --P 4 2>&1 | tail -1; done
