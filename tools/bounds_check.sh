#!/bin/bash
# Debug-bounds build (every shared-memory scatter / slot / hash index checked,
# a violation traps) run over the sanitizer smoke and the GPU test suite; the
# stand-in for compute-sanitizer, which this GPU pool does not allow.
# Build here: tools/bounds_check.sh build ; run under gpurun: tools/bounds_check.sh run
set -u
cd "$(dirname "$0")/.."
if [ "${1:-run}" = build ]; then
  mkdir -p build/debug
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -shared -Xcompiler -fPIC \
       -DFPSSFT_DEBUG_BOUNDS=1 -o build/debug/libfpssft.so paper_1711_11407_b200/csrc/fpssft.cu
  exit $?
fi
O=gpurun_out/bounds
mkdir -p $O
FPSSFT_LIB=build/debug/libfpssft.so timeout 600 python tools/sanitize_smoke.py > $O/smoke.txt 2>&1
echo "rc=$?" >> $O/smoke.txt
FPSSFT_LIB=build/debug/libfpssft.so timeout 1200 python -m pytest tests -m gpu -q -x > $O/tests.txt 2>&1
echo "rc=$?" >> $O/tests.txt
FPSSFT_LIB=build/debug/libfpssft.so timeout 900 python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 3 --load-seconds 0 > $O/bench_c2.txt 2>&1
echo "rc=$?" >> $O/bench_c2.txt
FPSSFT_LIB=build/debug/libfpssft.so timeout 900 python bench.py --config 5 --batch 2048 --no-e2e --no-cpu-baseline --steps 2 --warmup 3 --load-seconds 0 > $O/bench_c5.txt 2>&1
echo "rc=$?" >> $O/bench_c5.txt
grep -h "FPSSFT_CHECK\|rc=" $O/*.txt
