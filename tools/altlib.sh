# build libswe_b200.so variants with extra nvcc defines into paper_2306_09497_b200/_build/<name>/
#   bash tools/altlib.sh <name> "-DFOO=1 -DBAR=2"     (A/B with SWE_LIB=... tools/pathbench.py)
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
D=$R/paper_2306_09497_b200/_build/$1
mkdir -p $D
for f in plan legendre legendre_v2 legendre_v3 fft fft_lanes spectral stepper diag settls; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xptxas -v \
    --expt-relaxed-constexpr -I $R/include $2 -c $R/paper_2306_09497_b200/csrc/$f.cu -o $D/$f.o > $D/$f.log 2>&1 || echo "FAILED $f (see $D/$f.log)" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static $D/*.o -o $D/libswe_b200.so
echo $D/libswe_b200.so
