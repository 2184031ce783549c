cd "$GRAFT_REPO_ROOT"
for v in ${VARIANTS:-ns6 ns4}; do for ps in ${PER_SM:-6 1}; do
  echo "== $v per_sm=$ps"; RK_LIB=alt/$v.so RK_VOTE_PER_SM=$ps timeout 300 python scripts/coschedule_probe.py 2>&1 | tail -4
done; done
