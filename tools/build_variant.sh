#!/bin/bash
# Build an experimental libvsbp.so variant with extra nvcc defines into exp/:
#   tools/build_variant.sh NAME -DFOO=1 -DBAR=2
# (run here; the .so travels with the gpurun snapshot; select with VSBP_LIB=exp/libvsbp_NAME.so)
set -e
NAME=$1; shift
mkdir -p exp/obj_$NAME
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 -Xptxas -O3"
pids=()
for f in paper_1902_09733_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc $FL "$@" -I include -I paper_1902_09733_b200/csrc -c $f -o exp/obj_$NAME/$(basename $f).o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o exp/libvsbp_$NAME.so exp/obj_$NAME/*.o
rm -rf exp/obj_$NAME
echo exp/libvsbp_$NAME.so
