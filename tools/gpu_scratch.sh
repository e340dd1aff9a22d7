for n in 8 16; do python tools/gap_probe.py 30720 $n 20; python tools/gap_probe.py 30720 $n 20 det; done
python tools/gap_probe.py 8192 8 50; python tools/gap_probe.py 8192 8 50 det
