#!/bin/bash
# Time config-3 stage splits for the product build and every exp/lib_*.so
# variant (tools/build_variant.sh):  tools/gpu/variants.sh [queries] [config]
Q=${1:-20000000}; C=${2:-3}
echo "== product"; python tools/profile_step.py --config $C --queries $Q --reps 3 2>&1 | tail -2
for f in exp/lib_*.so; do echo "== $f"; TCCD_LIB=$f python tools/profile_step.py --config $C --queries $Q --reps 3 2>&1 | tail -2; done
