# Build a variant of libgdb200.so with extra compile-time knobs for A/B runs
# (tools/gpu_variants.sh):  bash tools/build_variant.sh NAME "-DKNOB=1 ..."
set -e
name=$1; shift
here=$(cd "$(dirname "$0")/.." && pwd)
obj=/tmp/gdvar_$name
mkdir -p "$obj" "$here/variants"
make -s -j8 -C "$here/paper_2507_11094_b200/csrc" OBJDIR="$obj" OUT="$here/variants/libgdb200_$name.so" \
  EXTRA="$*" "$here/variants/libgdb200_$name.so"
echo "built variants/libgdb200_$name.so ($*)"
