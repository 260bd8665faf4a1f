#!/bin/sh
# Build locally, and only if that succeeds run the given command on the GPU box.
cd "$(dirname "$0")/.." || exit 1
./tools/build.sh > /tmp/b2_build.log 2>&1 || { grep -i error /tmp/b2_build.log | head; exit 1; }
(cd tools/tc_probe && make -s probe probe_skipa > /tmp/b2_probe_build.log 2>&1) || { grep -i error /tmp/b2_probe_build.log | head; exit 1; }
timeout "${GPU_TIMEOUT:-1800}" /usr/local/graft/bin/gpurun --timeout "${GPU_LIMIT:-600}" -- "$1"
