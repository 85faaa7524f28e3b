#!/usr/bin/env bash
# Clock-independent A/B of kernel variants: per-CTA cycles per kept tile of the dQ and dK/dV
# kernels (and the forward's per-SM ns/tile) from -DSPA2_CTA_TIMES builds.  Each argument is
# "name flags...", built here with tools/build_alt.sh; run the printed command on the GPU box.
#   bash tools/ab_cycles.sh "base" "p3 -DSPA2_DKDV_NQ=3"  -> builds alt/ct_base, alt/ct_p3
set -eu
CMD=""
for a in "$@"; do
  set -- $a; n=$1; shift
  bash "$(dirname "$0")/build_alt.sh" "ct_$n" -DSPA2_CTA_TIMES "$@" > /dev/null
  CMD="$CMD echo == $n; python tools/cta_times.py alt/ct_$n/libspa2.so | grep -E 'cycles per tile|== k_|SM clock';"
done
echo "$CMD"
