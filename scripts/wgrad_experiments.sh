# conv2 passes at P = 1, 2, 4, 8 (development aid)
cd $GRAFT_REPO_ROOT
pb() { timeout 60 python scripts/pass_bench.py --reps 10 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['variant']['P'], {k: round(v,4) for k,v in d['ms'].items()}, {k: round(v) for k,v in d['tflops'].items()})"; }
for P in 1 2 4 8; do pb --P $P; done
