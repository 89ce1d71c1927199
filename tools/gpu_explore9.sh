TACOS_TRACE_STRIDE=20 QS=4 timeout 600 python tools/trace_phases.py 4
QS=2 timeout 300 python tools/trace_phases.py 3
