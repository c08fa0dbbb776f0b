# Full tree of a commit (default HEAD) with its library built, under tools/exp/tree_<name>/, for
# A/B runs across ABI changes:  (cd tools/exp/tree_<name> && python tools/ab.py)
set -e
REV=${1:-HEAD}; NAME=${2:-head}
R=$(git rev-parse --show-toplevel)
D=$R/tools/exp/tree_$NAME
rm -rf "$D"; mkdir -p "$D"
git -C "$R" archive "$REV" | tar -x -C "$D"
(cd "$D" && python -c "from paper_1511_03645_b200 import build as b; b.build()" > /dev/null)
echo built "$D"
