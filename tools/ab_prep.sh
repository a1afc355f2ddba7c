# tools/ab_prep.sh <name> [experiment bits]: copy the current package to ab/<name>
# and build it there, optionally with -DGJ_UMMA_EXPERIMENT=<bits> (timing
# experiments of the tcgen05 join, gj_join_umma.cu).  ab/ is git-ignored but
# ships to the GPU box with gpurun; time two copies with tools/ab_join.py.
set -e
v=$1
bits=${2:-0}
rm -rf ab/$v && mkdir -p ab/$v
cp -r paper_1809_09930_b200 include ab/$v/
rm -rf ab/$v/paper_1809_09930_b200/build ab/$v/paper_1809_09930_b200/__pycache__ ab/$v/paper_1809_09930_b200/libgpujoin.so
(cd ab/$v && GJ_NVCC_EXTRA="-DGJ_UMMA_EXPERIMENT=$bits ${GJ_NVCC_EXTRA:-}" python -c "import sys; sys.path.insert(0,'.'); import importlib; print(importlib.import_module('paper_1809_09930_b200._build').build(force=True))")
