#!/bin/bash
# Build libtpl.so of a git revision into paper_1812_01108_b200/build/libtpl_<name>.so for
# same-box A/B runs (TPL_LIB=<that path> python bench.py ...):  tools/ab_build.sh REV [name]
set -e
cd "$(dirname "$0")/.."
REV=${1:-HEAD}; NAME=${2:-base}
WT=/tmp/tpl_ab_$NAME
rm -rf "$WT"; git worktree prune
git worktree add -f --detach "$WT" "$REV" > /dev/null
(cd "$WT" && python paper_1812_01108_b200/build.py --force > /dev/null)
mkdir -p paper_1812_01108_b200/build
cp "$WT/paper_1812_01108_b200/libtpl.so" "paper_1812_01108_b200/build/libtpl_$NAME.so"
git worktree remove --force "$WT"
echo "paper_1812_01108_b200/build/libtpl_$NAME.so"
