#!/bin/bash
# A/B experiments of compile-time variants: recompile the listed csrc/*.cu with extra nvcc flags
# and link them with the other objects of build/ into OUT (load it with FDPD_LIB=OUT).
# usage: tools/build_variant.sh OUT.so "-DFOO=1" chain_cl.cu [tx.cu ...]
set -e
OUT=$1; DEFS=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
VB=$(mktemp -d)
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="$ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -cudart static --expt-relaxed-constexpr"
for f in "$@"; do nvcc $FLAGS $DEFS -c "$ROOT/paper_2205_05158_b200/csrc/$f" -o "$VB/${f%.cu}.o"; done
OBJS=""
for o in "$ROOT"/build/*.o; do b=$(basename "$o"); [ -f "$VB/$b" ] && OBJS="$OBJS $VB/$b" || OBJS="$OBJS $o"; done
nvcc $ARCH -shared -cudart static -o "$OUT" $OBJS
echo "built $OUT"
