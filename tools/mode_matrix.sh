#!/bin/bash
# timing matrix of the operator kernels at 1024^2 Q2 (configs[1] inputs)
for sp in miehe none; do for g in 0 1; do for md in 0 1 2 3; do
  python tools/prof_apply.py --split $sp --mode $md --reps 20 --generic $g 2>/dev/null | sed "s/^/generic=$g /"
done; done; done
