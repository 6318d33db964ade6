#!/bin/bash
# full ncu capture of k_cycle of the default build (tag $1)
bash tools/prof_k.sh k_cycle ${1:-kc_new}
exit 0
