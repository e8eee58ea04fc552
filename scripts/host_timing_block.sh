#!/bin/bash
# Host-side checkpoints of run_vqe on the shared-memory engine
# (-DVQF_HOST_TIMING build in /tmp), n given as arguments.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/vqf_ht && mkdir -p /tmp/vqf_ht
cp -r "$ROOT/paper_2601_09951_b200" "$ROOT/include" "$ROOT/scripts" "$ROOT/tools" /tmp/vqf_ht/
cd /tmp/vqf_ht/paper_2601_09951_b200/csrc
sed -i 's/^FLAGS := $(ARCH)/FLAGS := -DVQF_HOST_TIMING $(ARCH)/' Makefile
rm -rf build/vqe_host.o ../libvqf_b200.so && make -j8 >/dev/null 2>&1
cd /tmp/vqf_ht && python scripts/block_probe.py "$@" "$@" "$@" 2>&1 | tail -24
