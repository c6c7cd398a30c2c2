#!/bin/bash
cd $(dirname $0)/../..
bash tools/ab.sh "skp allwait" "cfg2 sweep1024 gsweep2048 sweep8192 cfg3 circ1024" 2
