# r02 call C: end-to-end time breakdown, a config-3 knob check, then compute-sanitizer memcheck on small cases.
python -c "from paper_2304_05301_b200 import build; build.build()"
python tools/host_breakdown.py 3 > gpurun_out/r02c_host_breakdown_c3.txt 2>&1; cat gpurun_out/r02c_host_breakdown_c3.txt
for wlst in 0 1; do TACOS_WORKLIST=$wlst python tools/time_search.py 3 0 20; done > gpurun_out/r02c_knobs_c3.txt 2>&1; cat gpurun_out/r02c_knobs_c3.txt
python tools/sanitize_cases.py > gpurun_out/r02c_sanitize_plain.txt 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 python tools/sanitize_cases.py > gpurun_out/r02c_memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -15 gpurun_out/r02c_memcheck.txt
