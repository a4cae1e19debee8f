# Build libsrt from the working tree with some files taken from another git
# revision, into abtest/libsrt_<tag>.so (development A/B timing: load it with
# SRT_LIB=abtest/libsrt_<tag>.so; extra nvcc flags in $NVFLAGS).
# Usage: bash tools/build_ab.sh <tag> <rev> <file>...
set -e
TAG=$1; REV=$2; shift 2
W=/tmp/ab_$TAG; rm -rf $W; mkdir -p $W/pkg $W/include
cp -r paper_2601_09083_b200/csrc $W/pkg/; cp include/srt.h $W/include/
for f in "$@"; do git show $REV:paper_2601_09083_b200/csrc/$f > $W/pkg/csrc/$f; done
cd $W/pkg/csrc
for f in *.cu; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false -Xcompiler -fPIC -Xcompiler -fvisibility=hidden $NVFLAGS -c $f -o $W/${f%.cu}.o & done; wait
cd - > /dev/null; mkdir -p abtest
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o abtest/libsrt_$TAG.so $W/*.o -lcudart
echo abtest/libsrt_$TAG.so
