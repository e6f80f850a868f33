# Build A/B variants of libbsa.so into csrc/build/<name>/ (kernel experiments).
# usage: scripts/build_variants.sh name1:"-DFOO=1" name2:"-DBAR=2" ...
set -e
cd "$(dirname "$0")/../paper_2509_07120_b200/csrc"
for spec in "$@"; do
  name="${spec%%:*}"; defs="${spec#*:}"
  out=build/$name; mkdir -p $out
  for f in ${BSA_VARIANT_FILES:-bsa_capi bsa_score bsa_scoresel bsa_attn_simt bsa_attn_tc bsa_attn_host bsa_stats_tc bsa_qkv_tc}; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      -diag-suppress 550,128,177 -I../../include $defs -c $f.cu -o $out/$f.o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libbsa.so $out/*.o
done
