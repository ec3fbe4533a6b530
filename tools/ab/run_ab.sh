#!/bin/bash
# A/B: tools/ab/libstrom_base.so (previous build) vs the in-tree libstrom.so
set -x
python tools/quick_time.py 2>&1 | grep -E "us/iter|^\[" 
STROM_LIB=$PWD/tools/ab/libstrom_base.so python tools/quick_time.py 2>&1 | grep -E "us/iter|^\["
python tools/shapes_time.py cartpole:30 2>&1 | cut -c1-200
STROM_LIB=$PWD/tools/ab/libstrom_base.so python tools/shapes_time.py cartpole:30 2>&1 | cut -c1-200
