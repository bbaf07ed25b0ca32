# time cfg3 with several tuning builds: bash tools/sweep_libs.sh name1 name2 ... ("" = product lib)
for n in "$@"; do
  if [ "$n" = "release" ]; then L=""; else L="paper_1608_04431_b200/libfa_$n.so"; fi
  echo "== $n"
  FA_LIB=$L python tools/sweep.py ${CFG:-cfg3} 0 "BR=32;BR=32" 2>&1 | tail -2
done
