# Build the committed HEAD's library into tools/exp/lib_head.so (A/B baseline for ab.py).
set -e
R=$(git rev-parse --show-toplevel)
D=$(mktemp -d)
git -C "$R" archive HEAD paper_1511_03645_b200 include | tar -x -C "$D"
python -c "import sys; sys.path.insert(0, '$D'); from paper_1511_03645_b200 import build as b; b.build(lib='$R/tools/exp/lib_head.so', build_dir='$D/_b')"
rm -rf "$D"
echo built tools/exp/lib_head.so
