#!/bin/bash
cd "$GRAFT_REPO_ROOT"
bash tools/c3_variants.sh $1
