for w in sweep2048 gsweep2048 sweep4096 gsweep4096 sweep8192 gsweep8192; do
STEPS=200 bash tools/variant.sh run "main e1u1 e1u2" $w 2>&1
done
