#!/bin/bash
# Build the committed HEAD's library as _lib/libbsccs_b200_<name>.so (A/B
# against the working tree's build; scripts/ab_rcd.sh picks up every variant).
set -e
name=${1:-xold}
cp paper_1208_0945_b200/_lib/libbsccs_b200.so /tmp/_wt.so
git stash -q
python -c "import sys; sys.path.insert(0,'.'); from paper_1208_0945_b200 import build as b; b.build_native()" 2>&1 | grep -E "error" || true
cp paper_1208_0945_b200/_lib/libbsccs_b200.so paper_1208_0945_b200/_lib/libbsccs_b200_$name.so
git stash pop -q
cp /tmp/_wt.so paper_1208_0945_b200/_lib/libbsccs_b200.so
touch paper_1208_0945_b200/csrc/*.cu
