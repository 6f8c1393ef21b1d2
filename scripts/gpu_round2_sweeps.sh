#!/bin/bash
# GPU session: paper sweeps (scripts/paper_sweeps.py).  First a Gram-vs-QR compressor check at n = 64.
cd "$GRAFT_REPO_ROOT"
FMMT_COMPRESS_GRAM=1 timeout 900 python scripts/paper_sweeps.py E1 --max-n 64 --out gpurun_out/sweep_gram_check.jsonl > gpurun_out/sweep_gram_check.log 2>&1; echo "gram check rc=$?"
timeout 2400 python scripts/paper_sweeps.py E1 --max-n 256 --out gpurun_out/paper_sweeps.jsonl > gpurun_out/sweep_E1.log 2>&1; echo "E1 rc=$?"
timeout 1800 python scripts/paper_sweeps.py E3 --max-n 256 --out gpurun_out/paper_sweeps.jsonl > gpurun_out/sweep_E3.log 2>&1; echo "E3 rc=$?"
