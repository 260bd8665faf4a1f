#!/bin/sh
# Build the sm_100a library (and the oracle) without importing the package.
cd "$(dirname "$0")/.." && python -c "import __graft_entry__ as g; g.build()"
