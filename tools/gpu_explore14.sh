TACOS_TRACE_STRIDE=20 QS=8 timeout 600 python tools/trace_phases.py 4
