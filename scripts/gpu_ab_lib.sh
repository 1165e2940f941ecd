# A/B: variants/old.so (previous build) vs the tree's build, C2 step kernel times (scripts/ab_step.py)
for i in 1 2 3; do
  echo -n "old: "; CKO_LIB_PATH=variants/old.so PYTHONPATH=. timeout 300 python scripts/ab_step.py 5
  echo -n "new: "; PYTHONPATH=. timeout 300 python scripts/ab_step.py 5
  echo -n "new fused: "; PYTHONPATH=. timeout 300 python scripts/ab_step.py 5 fused
done
