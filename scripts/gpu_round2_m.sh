#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python scripts/mem_probe.py tucker3d:8 tucker3d:32 tt3d:8 tt3d:32 tt4d:435 tucker4d:435 htucker4d:435 tucker3d:435 > gpurun_out/mem_probe_m.log 2>&1; echo "probe rc=$?"
tail -30 gpurun_out/mem_probe_m.log
