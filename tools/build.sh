#!/bin/bash
# Build the C-ABI library in-tree (same as __graft_entry__.build()).
cd "$(dirname "$0")/.." && python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('b', 'paper_2304_09770_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build()"
