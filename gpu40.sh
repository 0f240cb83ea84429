cd $GRAFT_REPO_ROOT
for pad in 0 8704 0 8704; do
  echo "pad=$pad"; HX_SK_SMEM_PAD=$pad timeout 600 python tools/ablate_step.py 2>&1 | grep -E "^none|all-but"
done
