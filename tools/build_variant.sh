#!/bin/bash
# Builds a variant of libbbcodec.so with one source recompiled under extra -D flags.
#   tools/build_variant.sh NAME SOURCE.cu -DKNOB=VALUE ...   ->  _variants/NAME.so
# The other objects come from the regular in-tree build (run `make` in csrc first).
# Knobs: PF_B1 PF_B2 PF_THREADS_OVR BK_THREADS_OVR K5_G_BIG K5_PT HP7_TP HP7_W_OVR HP4_SEG_OVR
#        (bb_deflate.cu); WD_WARPS_OVR ND_THREADS_OVR RS_THREADS_OVR DS_MINB RC_THREADS VD_THREADS
#        VD_GRID_MUL (bb_inflate_par.cu).
set -e
name=$1; src=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
cd "$root/paper_2604_21072_b200/csrc"
tmp=$(mktemp -d)
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -I../../include "$@" -dc -o "$tmp/${src%.cu}.o" "$src" 2>/dev/null
objs=""
for o in build/*.o; do
  if [ "$(basename "$o")" = "${src%.cu}.o" ]; then objs="$objs $tmp/${src%.cu}.o"; else objs="$objs $o"; fi
done
mkdir -p "$root/_variants"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/_variants/$name.so" $objs -lcudart
rm -rf "$tmp"
echo "built _variants/$name.so"
