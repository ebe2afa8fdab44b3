#!/bin/bash
# A/B builds: tools/mk_ab.sh NAME [extra nvcc flags...] → ab/NAME/paper_2101_07948_b200 (package + libsdnn.so)
set -e
name=$1; shift
rm -rf ab/$name && mkdir -p ab/$name
cp -r paper_2101_07948_b200 include ab/$name/
rm -f ab/$name/paper_2101_07948_b200/libsdnn.so
SDNN_NVCC_FLAGS="$*" python -c "
import importlib.util,sys
spec=importlib.util.spec_from_file_location('b','ab/$name/paper_2101_07948_b200/build.py'); m=importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)"
ls -la ab/$name/paper_2101_07948_b200/libsdnn.so
