#!/bin/bash
# Build A/B variants of librsa_b200.so into tools/ab_so/<name>.so:
#   tools/build_variants.sh name1 "-DFOO=1 -DBAR=2" name2 "-DFOO=3" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/ab_so
cp paper_2511_19835_b200/librsa_b200.so /tmp/librsa_keep.so
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  rm -rf paper_2511_19835_b200/_build_ab
  RSA_EXTRA_NVCC="$flags" python - <<PY
import paper_2511_19835_b200.build as b, shutil
from pathlib import Path
b.OBJ = b.PKG / "_build_ab"
b.LIB = Path("tools/ab_so/$name.so").resolve()
b.build(verbose=False)
PY
  echo "built $name ($flags)"
done
cp /tmp/librsa_keep.so paper_2511_19835_b200/librsa_b200.so
