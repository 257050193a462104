#!/bin/bash
# k_mc variants side by side (bench lines with phase times).  scripts/r2h_ab.sh TAG
export NOTEST=1
LIBS="${LIBS:-default mom6 mb5 mom6mb5}" CONFIGS="${CONFIGS:-C3f C1}" bash scripts/r2e_ab.sh ${1:-r2h}
