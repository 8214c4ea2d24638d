# Builds the library with extra nvcc flags into abl/<name>.so for A/B runs
# (scripts/ab_kernels.py), from a copy of the working tree:
#   bash scripts/build_variant.sh <name> "-DFLAG ..."
set -e
name=$1
flags=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
cp -r "$root/paper_2403_13287_b200" "$root/include" "$tmp/"
rm -rf "$tmp/paper_2403_13287_b200/csrc/build" "$tmp/paper_2403_13287_b200/liblskum_b200.so"
make -s -C "$tmp/paper_2403_13287_b200/csrc" -j16 NVEXTRA="$flags"
mkdir -p "$root/abl"
cp "$tmp/paper_2403_13287_b200/liblskum_b200.so" "$root/abl/$name.so"
grep -A3 "k_flux_wsILi2ELi8ELi5\|k_sweep_tile" "$tmp/paper_2403_13287_b200/csrc/build/ptxas.log" | grep -E "registers|spill" | head -4
rm -rf "$tmp"
