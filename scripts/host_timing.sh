#!/bin/bash
# Host-side checkpoints of one run_sweep call (-DVQF_HOST_TIMING build in /tmp).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/vqf_ht && mkdir -p /tmp/vqf_ht
cp -r "$ROOT/paper_2601_09951_b200" "$ROOT/include" "$ROOT/scripts" "$ROOT/tools" /tmp/vqf_ht/
cd /tmp/vqf_ht/paper_2601_09951_b200/csrc
sed -i 's/^FLAGS := $(ARCH)/FLAGS := -DVQF_HOST_TIMING $(ARCH)/' Makefile
rm -rf build ../libvqf_b200.so && make -j8 >/dev/null 2>&1
cd /tmp/vqf_ht && E2E_NOTRAJ=1 python scripts/e2e_breakdown.py 20 2>&1 | tail -30
