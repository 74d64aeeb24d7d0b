# forward pass time at P=1/2/4 on the default build (regression check)
for P in 1 2 4; do
  echo "P=$P $(timeout 100 python scripts/pass_bench.py --P $P --reps 20 2>&1 | tail -1 | grep -o '"fwd": [0-9.]*' | head -1)"
done
