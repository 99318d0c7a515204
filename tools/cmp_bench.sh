# A/B: the current tree against worktrees of earlier commits (same box, back to back)
for d in . .cmp_old2 .cmp_old . .cmp_old2 .cmp_old; do
  (cd $d && python bench.py --no-cpu-baseline --steps 5 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$d', j['roofline']['achieved'])")
done
