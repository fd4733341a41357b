# Build a variant of libgesr.so with extra nvcc flags:  scripts/mkvar.sh NAME "-DFOO -DBAR"
# [SRC_DIR]: optional csrc copy (e.g. an older revision).
# -> build/ab/NAME.so (A/B with scripts/ab.sh; GESR_LIB selects the library).
set -e
rm -rf build/v_$1
name=$1; flags=$2
out=build/v_$name; mkdir -p $out build/ab
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I$PWD/include -I$PWD/paper_2511_21095_b200/csrc $flags"
S=${3:-paper_2511_21095_b200/csrc}
for f in proj attn attn2 hma stu nro debug hostpath; do $NV -c $S/$f.cu -o $out/$f.o & done
$NV -x cu -c $S/capi.cpp -o $out/capi.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/ab/$name.so \
  $out/proj.o $out/attn.o $out/attn2.o $out/hma.o $out/stu.o $out/nro.o $out/debug.o $out/hostpath.o $out/capi.o -Xlinker --version-script=$S/exports.map
echo built build/ab/$name.so
