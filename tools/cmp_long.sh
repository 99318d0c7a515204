# A/B of the long kernel: current tree against an earlier worktree, back to back
for d in . .cmp_old . .cmp_old; do
  (cd $d && python tools/long_blocks.py 5000000 0 2>&1 | tail -1 | sed "s|^|$d |")
done
