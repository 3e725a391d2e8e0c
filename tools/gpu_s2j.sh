cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python tools/ws_parts.py cfg5 2,3 0,1,2,3 2>&1 | grep cfg
