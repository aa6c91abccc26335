for split in miehe none; do for cr in 0 1; do for rows in 0 16 24 32 40 64; do
  echo -n "split=$split CR=$cr rows=$rows: "; PFF_SWEEP_COLRING=$cr timeout 100 python tools/prof_apply.py --split $split --rows $rows --reps 50 2>&1 | tail -1
done; done; done
