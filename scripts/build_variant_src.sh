# Builds a libvqf_b200.so variant into _variants/<name>.so (git-ignored) with
# one object replaced by <src.cu> compiled with the Makefile's flags, e.g.
#   bash scripts/build_variant_src.sh expold /tmp/expold/expect_tile.cu expect_tile
set -e
name=$1; src=$2; obj=$3; shift 3
C=paper_2601_09951_b200/csrc
mkdir -p _variants/$name.obj
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-O2 -Iinclude -I$C \
  -Xptxas -v "$@" -c $src -o _variants/$name.obj/$obj.o 2> _variants/$name.ptxas.log
objs=$(ls $C/build/*.o | grep -v "/$obj.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/$name.so $objs _variants/$name.obj/$obj.o -lpthread
echo "built _variants/$name.so"
