#!/bin/sh
# Build the sm_100a library in-tree (also done by __graft_entry__.build()).
set -e
cd "$(dirname "$0")"
python -c "import paper_1307_2895_b200._build as b; b.build(verbose=True)"
