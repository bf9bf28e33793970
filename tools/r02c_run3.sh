#!/bin/bash
set -u
CFGS="c5" bash tools/r02_prof.sh
SETS="RADSORT_LOCAL_WDELTA=0|RADSORT_LOCAL_WDELTA=-1|RADSORT_LOCAL_WDELTA=1" CFGS="c4 c5" bash tools/r02c_envab.sh
