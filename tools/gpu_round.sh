set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for c in fma dmma ffma2; do TSM2X_CONSUMER=$c timeout 300 python tools/quickbench.py --impls tma --configs r8,r16,f16,l16 2>&1 | sed "s/^/$c /"; done
timeout 600 python tools/quickbench.py --sustain 2>&1 | tail -20
TSM2X_CONSUMER=fma timeout 600 python tools/quickbench.py --sustain 2>&1 | tail -20 | sed "s/^/fma /"
