#!/bin/bash
cd $(dirname $0)/../..
bash tools/ab.sh "skp split" "cfg2 sweep1024 gsweep2048 gsweep4096 sweep8192 circ1024 cfg4" 2
