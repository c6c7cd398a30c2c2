for r in 1 2; do for w in sweep2048 gsweep2048 sweep4096 gsweep4096; do
STEPS=200 bash tools/variant.sh run "main nokfs slotwg" $w 2>&1
done; done
