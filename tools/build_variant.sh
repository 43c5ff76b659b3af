# Build an A/B variant of the library with extra nvcc defines:
#   bash tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"   ->  build/NAME/libb200fd.so
set -e
NAME=$1; DEFS=$2
NV="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC"
mkdir -p build/$NAME
for s in paper_1608_03984_b200/csrc/*.cu; do
  b=$(basename $s .cu)
  nvcc $NV $DEFS -c -o build/$NAME/$b.o $s &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/$NAME/libb200fd.so build/$NAME/*.o
echo built build/$NAME/libb200fd.so
