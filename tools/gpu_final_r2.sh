#!/bin/bash
# Final round-2 capture: the evidence script, then the GPU suite on the
# bounds-asserting build and the conformance run.
bash tools/gpu_evidence_r2.sh
DARE_CHECKED=1 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/ev_pytest_gpu_checked.log 2>&1; echo "checked=$?" >> gpurun_out/ev_status.txt
bash tools/conformance.sh > gpurun_out/ev_conformance.log 2>&1; echo "conformance=$?" >> gpurun_out/ev_status.txt
cat gpurun_out/ev_status.txt
