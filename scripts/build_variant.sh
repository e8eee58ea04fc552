# Builds a libvqf_b200.so variant with extra nvcc flags for tile.cu into
# _variants/<name>.so (git-ignored), e.g.
#   bash scripts/build_variant.sh g4s1 -DVQF_TILE_GROUPS=4 -DVQF_TILE_STAGES=1
set -e
name=$1; shift
C=paper_2601_09951_b200/csrc
mkdir -p _variants/$name.obj
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-O2 -Iinclude -I$C \
  -Xptxas -v "$@" -c $C/tile.cu -o _variants/$name.obj/tile.o 2> _variants/$name.ptxas.log
objs=$(ls $C/build/*.o | grep -v "/tile.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/$name.so $objs _variants/$name.obj/tile.o -lpthread
echo "built _variants/$name.so"
