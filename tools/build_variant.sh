# build_variant.sh NAME "NVCC FLAGS" file.cu [file.cu ...]: relink libmapple_b200.so with the
# given sources recompiled under extra flags, into csrc/build/NAME/lib.so (for MAPPLE_B200_LIB A/Bs)
set -e
cd "$(dirname "$0")/../paper_2507_17087_b200/csrc"
name=$1; flags=$2; shift 2
out=build/$name; mkdir -p $out
objs=""
for o in build/*.o; do
  src=$(basename $o .o)
  skip=0; for f in "$@"; do [ "$src" = "$f" ] && skip=1; done
  [ $skip = 0 ] && objs="$objs $o"
done
for f in "$@"; do
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -O3 -Ibuild $flags -c $f -o $out/$f.o
  objs="$objs $out/$f.o"
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/lib.so $objs -L/usr/local/cuda/lib64 -lnvrtc -Xlinker -rpath,/usr/local/cuda/lib64
echo $out/lib.so
