#!/bin/bash
# Build an A/B variant of libchunkode_b200.so with extra -D flags for the
# per-model kernel files: scripts/build_variant.sh NAME "-DFOO=1 -DBAR=2"
# -> variants/NAME.so (load with CKO_LIB_PATH=variants/NAME.so).
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2310_08649_b200/csrc
OBJ=$ROOT/build/csrc
OUT=$ROOT/variants/$NAME
mkdir -p "$OUT"
make -s -C "$SRC" >/dev/null
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
OBJS=""
for f in "$OBJ"/*.o; do
  b=$(basename "$f" .o)
  case $b in
    cko_inst_*) nvcc $FLAGS $DEFS -c "$SRC/$b.cu" -o "$OUT/$b.o" & OBJS="$OBJS $OUT/$b.o" ;;
    *) OBJS="$OBJS $f" ;;
  esac
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared $OBJS -o "$ROOT/variants/$NAME.so" -lcudart -lpthread
rm -rf "$OUT"
echo "variants/$NAME.so"
