# fused scoring A/B: bit-identity vs the three-kernel path, launch shapes,
# phase-A-only timing (BSA_SCORESEL_DEBUG=1 skips phase B; results wrong)
python scripts/scoresel_ab.py 2>&1 | tail -15
for shape in 0 1; do for dbg in 0 1; do
  echo "shape $shape debug $dbg: $(BSA_SCORESEL_SHAPE=$shape BSA_SCORESEL_DEBUG=$dbg python scripts/scoresel_ab.py --arm /tmp/x.npz 2>&1 | head -1)"
done; done
