#!/bin/bash
cd "$GRAFT_REPO_ROOT"
bash tools/c2_variants.sh $1
