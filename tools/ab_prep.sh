# tools/ab_prep.sh: copy the current package to abtest/$1 and build it there (for tools/ab_join.py)
set -e
v=$1
rm -rf abtest/$v && mkdir -p abtest/$v
cp -r paper_1809_09930_b200 include abtest/$v/
rm -rf abtest/$v/paper_1809_09930_b200/build abtest/$v/paper_1809_09930_b200/__pycache__ abtest/$v/paper_1809_09930_b200/libgpujoin.so
(cd abtest/$v && python -c "import sys; sys.path.insert(0,'.'); import importlib; print(importlib.import_module('paper_1809_09930_b200._build').build(force=True))")
