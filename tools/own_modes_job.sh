timeout 500 python -u tools/own_modes.py
