#!/bin/bash
# Build the committed HEAD into tools/libjdob_prev.so (git worktree) for an A/B against the working tree.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/wt_prev && git worktree add -q /tmp/wt_prev HEAD
(cd /tmp/wt_prev && tools/build_variants.sh prev "" > /dev/null 2>&1)
cp /tmp/wt_prev/tools/libjdob_prev.so tools/
git worktree remove --force /tmp/wt_prev
