#!/bin/bash
# resident kernel timing with and without its grid barrier (the second gives wrong fields)
for lib in default nobar; do
  if [ $lib = default ]; then L=""; else L=$PWD/paper_1909_05098_b200/libfedheat_b200_$lib.so; fi
  FH_LIB=$L timeout 300 python scripts/resident_sweep.py cfg1 1000 2>&1 | head -3 | sed "s/^/$lib /"
done
