# per-chunk time vs ring depth (CTA-pair kernels): rebuild with CP_TC_STAGES_CG2=N and time the
# conv2 passes alone at P=1/4 (scripts/pass_bench.py); restores the default build at the end
for st in 6 5 4; do
  CP_NVCC_EXTRA="-DCP_TC_STAGES_CG2=$st" python -c "from paper_1712_02546_b200 import build; build.build(force=True)"
  for P in 1 4; do
    echo "stages=$st P=$P $(timeout 100 python scripts/pass_bench.py --P $P --reps 20 2>/dev/null | cut -c1-260)"
  done
done
python -c "from paper_1712_02546_b200 import build; build.build(force=True)"
