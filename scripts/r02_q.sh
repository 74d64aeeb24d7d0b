# conv1 forward B-set size (images per set) vs weight-ring depth
for v in "4 4" "2 4" "2 6" "2 8" "1 8"; do set -- $v
  CP_C1_NB=$1 CP_C1_ASTAGES=$2 timeout 300 python scripts/conv1_bench.py > gpurun_out/r02q_nb$1_a$2.jsonl 2>&1; echo "nb=$1 a=$2 rc=$?"
  python -c "
import json
for l in open('gpurun_out/r02q_nb$1_a$2.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['P'], round(d['new_ms']['fwd']*1e3,1), d['y_rel'], d['codes_diff'])"
done
