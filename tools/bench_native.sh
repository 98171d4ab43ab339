#!/bin/bash
# Build and run tools/bench_native.c (the hot path timed from plain C through the C ABI).
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
CUDA="${CUDA_HOME:-/usr/local/cuda}"
python -c "import sys; sys.path.insert(0, '$ROOT'); import inputs, paper_cs_0406049_b200 as sp; inputs.build(); sp.lib()"
gcc -O2 -std=c99 -D_GNU_SOURCE -o /tmp/bench_native "$ROOT/tools/bench_native.c" -I"$CUDA/include" \
    -L"$ROOT/paper_cs_0406049_b200" -L"$ROOT/inputs" -L"$CUDA/lib64" -lsincos_pairs -lsincos_inputs -lcudart \
    -Wl,-rpath,"$ROOT/paper_cs_0406049_b200:$ROOT/inputs:$CUDA/lib64"
[ "${1:-}" = "--build-only" ] || /tmp/bench_native "$@"
