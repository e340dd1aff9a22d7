# Sustained (power-capped) time, SM clock and instantaneous power of every BASELINE workload with
# its default consumer, plus the arithmetic-free pipeline (TSM2X_CONSUMER=null) for the fp64 and
# fp32 TSM2R shapes — the data behind the energy model in DESIGN.md §4. Run under gpurun:
#   bash tools/energy_table.sh > gpurun_out/energy.log
for cfg in r2 r4 r8 r16 l16 f8 f16; do
  python tools/envab.py --cfg $cfg --rounds 2 --cands "base" 2>&1 | grep "^$cfg"
done
python tools/envab.py --cfg r8 --rounds 2 --cands "TSM2X_CONSUMER=null" 2>&1 | grep "^r8"
python tools/envab.py --cfg f16 --rounds 2 --cands "TSM2X_CONSUMER=null" 2>&1 | grep "^f16"
python tools/envab.py --cfg l16 --rounds 2 --cands "TSM2X_CONSUMER=null" 2>&1 | grep "^l16"
