# A/B of variant libraries (tools/altlib.sh) on the cfg2 fine step: bash tools/ab_libs.sh <name>...
for rep in 1 2; do
for n in base "$@"; do
  if [ $n = base ]; then L=paper_2306_09497_b200/libswe_b200.so; else L=paper_2306_09497_b200/_build/$n/libswe_b200.so; fi
  echo "== $n $(SWE_LIB=$L python tools/pathbench.py fft_rm=2 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"class_ms": {[^}]*}')"
done; done
