python tools/matrix_copy_probe.py
