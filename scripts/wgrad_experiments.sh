# dgrad L2 policy hints A/B (development aid)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for h in 0 1; do for P in 1; do echo -n "hint=$h "; CP_TC_L2HINT=$h timeout 60 python scripts/pass_bench.py --reps 10 --P $P 2>&1 | tail -1; done; done; done
for P in 2 4; do for h in 0 1; do echo -n "hint=$h "; CP_TC_L2HINT=$h timeout 60 python scripts/pass_bench.py --reps 10 --P $P 2>&1 | tail -1; done; done
