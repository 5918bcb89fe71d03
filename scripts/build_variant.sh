# build a study variant of the library: bash scripts/build_variant.sh NAME -DFLAG=V ...
# -> paper_1904_01201_b200/_lib/variants/libnavsim_NAME.so (select with NAVSIM_B200_LIB)
N=$1; shift
mkdir -p paper_1904_01201_b200/_lib/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -shared \
  -Xcompiler -fPIC,-ffp-contract=off "$@" -o paper_1904_01201_b200/_lib/variants/libnavsim_$N.so \
  paper_1904_01201_b200/csrc/navsim_b200.cu
