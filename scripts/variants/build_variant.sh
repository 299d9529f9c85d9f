#!/bin/bash
# Build the library with extra nvcc defines into ab/<name>.so (A/B variants).
# usage: build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/../.."
name=$1; defs=$2
tmp=$(mktemp -d)
cp -r paper_2405_18328_b200 include $tmp/
rm -rf $tmp/paper_2405_18328_b200/_build $tmp/paper_2405_18328_b200/*.so
mkdir -p ab
(cd $tmp && WGP_NVCC_DEFS="$defs" PYTHONPATH=$tmp python -c "from paper_2405_18328_b200 import build as b; b.build(force=True)" > /dev/null)
cp $tmp/paper_2405_18328_b200/libwarmgp_b200.so ab/$name.so
rm -rf $tmp
echo "built ab/$name.so ($defs)"
