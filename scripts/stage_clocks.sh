#!/bin/bash
# Per-stage cycle budget of one H2 Adam iteration (bond 0, iteration 100):
# builds a -DVQF_STAGE_CLOCKS copy of the engine under /tmp and runs a PES.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/vqf_clk && mkdir -p /tmp/vqf_clk
cp -r "$ROOT/paper_2601_09951_b200" "$ROOT/include" "$ROOT/scripts" "$ROOT/tools" /tmp/vqf_clk/
cd /tmp/vqf_clk/paper_2601_09951_b200/csrc
sed -i "s/^FLAGS := \$(ARCH)/FLAGS := -DVQF_STAGE_CLOCKS ${EXTRA_FLAGS:-} \$(ARCH)/" Makefile
rm -rf build ../libvqf_b200.so && make -j8 >/dev/null 2>&1
cd /tmp/vqf_clk && python scripts/prof_targets.py pes 2>&1 | grep -E "STAGES|PROLOGUE|TIMELINE" > /tmp/stage.txt; grep -E "STAGES|PROLOGUE" /tmp/stage.txt | head -3; python3 scripts/timeline.py /tmp/stage.txt
