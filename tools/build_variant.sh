# Build an A/B variant of libsnmat.so with extra -D flags into
# paper_2305_02510_b200/libsnmat_<name>.so (out-of-tree objects under /tmp).
# usage: tools/build_variant.sh <name> -DFOO=1 -DBAR=2
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=/tmp/snb_variant_$name
rm -rf "$tmp" && mkdir -p "$tmp/paper_2305_02510_b200"
cp -r "$root/include" "$tmp/"
cp -r "$root/paper_2305_02510_b200/csrc" "$tmp/paper_2305_02510_b200/"
rm -rf "$tmp/paper_2305_02510_b200/csrc/build"
make -s -C "$tmp/paper_2305_02510_b200/csrc" -j16 \
  NVFLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I$tmp/paper_2305_02510_b200/csrc -I$tmp/include $*" \
  OUT="$root/paper_2305_02510_b200/libsnmat_$name.so"
