# fused scoring A/B: bit-identity vs the three-kernel path, cluster sizes,
# phase-A-only timing (BSA_SCORESEL_DEBUG=1 skips phase B; results wrong)
python scripts/scoresel_ab.py 2>&1 | tail -15
for c in 2 4 8; do for dbg in 0 1; do
  echo "cluster $c debug $dbg: $(BSA_SCORESEL_DEBUG=$dbg BSA_SCORESEL_CLUSTER=$c python scripts/scoresel_ab.py --arm /tmp/x.npz 2>&1 | head -1)"
done; done
