# A/B: variants/${AB_OLD:-head}.so (previous build) vs the tree's build, C2 step kernel times (scripts/ab_step.py)
OLD=${AB_OLD:-head}
[ -n "$AB_TESTS" ] && timeout 1200 python -m pytest $AB_TESTS -x -q -m gpu 2>&1 | tail -4
for i in 1 2 3; do
  echo -n "$OLD: "; CKO_LIB_PATH=variants/$OLD.so PYTHONPATH=. timeout 300 python scripts/ab_step.py 5 fused
  echo -n "new: "; PYTHONPATH=. timeout 300 python scripts/ab_step.py 5 fused
done
