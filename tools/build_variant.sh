# dev tool: build libmorea.so variants with extra -D flags into build/var/<name>.so
# usage: tools/build_variant.sh NAME SRCROOT [-DFOO=1 ...]
set -e
name=$1; root=$2; shift 2
out=build/var; mkdir -p $out
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC"
for s in morea_kernels morea_api; do
  /usr/local/cuda/bin/nvcc $F "$@" -I $root/include -I $root/paper_2303_04873_b200/csrc -c $root/paper_2303_04873_b200/csrc/$s.cu -o $out/$name.$s.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/$name.so $out/$name.morea_kernels.o $out/$name.morea_api.o
rm -f $out/$name.*.o
echo built $out/$name.so
