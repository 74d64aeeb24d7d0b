# forward per-chunk cost decomposition (timing only: CP_TC_DIAG makes results wrong):
# 1 = no MMAs, 2 = no A loads, 4 = no B loads; conv2 fwd alone at P=1/4 (needs the hook build)
CP_NVCC_EXTRA=-DCP_TC_DIAG_HOOK python -c "from paper_1712_02546_b200 import build; build.build(force=True)"
for P in 1 4; do
  for d in 0 1 2 4 6 3 5; do
    echo "P=$P diag=$d $(CP_TC_DIAG=$d timeout 100 python scripts/pass_bench.py --P $P --reps 20 2>&1 | tail -1 | grep -o '"fwd": [0-9.]*' | head -1)"
  done
done
