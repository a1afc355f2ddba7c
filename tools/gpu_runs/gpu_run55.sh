cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^(FAILED|E )|Error|error" | head -20
