#!/bin/bash
# Per-stage cycle budget of one shared-memory-engine iteration (CTA 0,
# iteration 2): builds a -DVQF_STAGE_CLOCKS copy of the library under /tmp
# and runs run_scaling_study at the given widths.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/vqf_bclk && mkdir -p /tmp/vqf_bclk
cp -r "$ROOT/paper_2601_09951_b200" "$ROOT/include" "$ROOT/scripts" "$ROOT/tools" /tmp/vqf_bclk/
cd /tmp/vqf_bclk/paper_2601_09951_b200/csrc
sed -i "s/^FLAGS := \$(ARCH)/FLAGS := -DVQF_STAGE_CLOCKS \$(ARCH)/" Makefile
rm -rf build/vqe_block.o ../libvqf_b200.so && make -j8 >/dev/null 2>&1
cd /tmp/vqf_bclk && python scripts/block_probe.py "$@" 2>&1 | grep BLOCK_STAGES
