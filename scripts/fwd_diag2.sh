CP_NVCC_EXTRA=-DCP_TC_DIAG_HOOK python -c "from paper_1712_02546_b200 import build; build.build(force=True)"
# MMA-only forward (CP_TC_DIAG=6: no TMA loads) vs N tile width at P=4: is the per-MMA time N-proportional?
for nw in 128 192 256; do
  echo "P=4 nw=$nw diag=6 $(CP_TC_FWD_NW=$nw CP_TC_DIAG=6 timeout 100 python scripts/pass_bench.py --P 4 --reps 20 2>&1 | tail -1 | grep -o '"fwd": [0-9.]*' | head -1)"
  echo "P=4 nw=$nw diag=0 $(CP_TC_FWD_NW=$nw timeout 100 python scripts/pass_bench.py --P 4 --reps 20 2>&1 | tail -1 | grep -o '"fwd": [0-9.]*' | head -1)"
done
for cg in 1; do
  echo "P=4 CTA_GROUP=1 diag=6 $(CP_TC_CTA_GROUP=1 CP_TC_DIAG=6 timeout 100 python scripts/pass_bench.py --P 4 --reps 20 2>&1 | tail -1 | grep -o '"fwd": [0-9.]*' | head -1)"
  echo "P=4 CTA_GROUP=1 diag=0 $(CP_TC_CTA_GROUP=1 timeout 100 python scripts/pass_bench.py --P 4 --reps 20 2>&1 | tail -1 | grep -o '"fwd": [0-9.]*' | head -1)"
done
