#!/bin/bash
# A/B the device throughput of library variants: bash scripts/ab.sh name1 name2 ... (lib/<name>.so; "default" = libwsgpu.so)
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = default ]; then python scripts/quickbench.py; else WSGPU_LIB=paper_2409_03365_b200/lib/$v.so python scripts/quickbench.py; fi
  done
done
