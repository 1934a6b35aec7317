#!/bin/bash
# build the library; print the error tail on failure
python paper_2211_16479_b200/build.py "$@" > /tmp/build.log 2>&1 && tail -1 /tmp/build.log || { grep -E "error|Error" -A3 /tmp/build.log | head -40; exit 1; }
