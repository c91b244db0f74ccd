#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 120 ./tools/tma_ingest_probe > $O/tma_ingest.txt 2>&1
