for P in 4 8; do CP_TC_PLAN_LOG=1 CP_TC_FWD_T=1 CP_TC_FWD_MC=1 timeout 90 python scripts/pass_bench.py --P $P --reps 3 2>&1 | grep "tc_fwd" | sort | uniq -c; done
