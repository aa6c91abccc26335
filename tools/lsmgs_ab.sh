# A/B of the low-sync MGS partials row count (side builds libpff_b200_rows{2,6,8}.so)
for lib in libpff_b200.so libpff_b200_rows2.so libpff_b200_rows6.so libpff_b200_rows8.so; do
  echo "== $lib"
  PFF_LIB=$PWD/paper_2005_00331_b200/$lib python tools/bench_ortho.py 2>&1 | grep lowsync
  PFF_LIB=$PWD/paper_2005_00331_b200/$lib python tools/prof_newton.py 2>&1 | grep -E "device total|lsmgs"
done
