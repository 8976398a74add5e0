cd $GRAFT_REPO_ROOT
for v in ${VARIANTS}; do
  echo "== $v"; STMG_ROOT=$GRAFT_REPO_ROOT/exp/$v timeout 300 python scripts/time_ops.py ${TW:-C5-128 C4} 2>&1 | tail -3
done
