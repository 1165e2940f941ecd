# A/B of library builds on the C2 step kernel times (scripts/ab_step.py, fused training-step call):
# AB_LIBS="head nofuse" compares variants/<name>.so with the tree's build ("new").
[ -n "$AB_TESTS" ] && timeout 1200 python -m pytest $AB_TESTS -x -q -m gpu --timeout 120 2>&1 | tail -4
for i in $(seq ${AB_ROUNDS:-3}); do
  for v in ${AB_LIBS:-head}; do
    echo -n "$v: "; CKO_LIB_PATH=variants/$v.so PYTHONPATH=. timeout 300 python scripts/ab_step.py 5 fused
  done
  echo -n "new: "; PYTHONPATH=. timeout 300 python scripts/ab_step.py 5 fused
done
