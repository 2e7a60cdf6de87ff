# e2e staging diagnostics: pinned-ness of the host queries, copy timeline per chunk size
DADE_GPU_VERBOSE=1 DADE_GPU_TIMELINE=1 python tools/e2e_breakdown.py 2>&1 | grep -E "host queries|host-buffer search|H2D" | sort | uniq -c | head
for c0 in 2048 3008 4096; do echo "CHUNK0=$c0"; DADE_GPU_CHUNK0=$c0 DADE_GPU_TIMELINE=1 python tools/e2e_breakdown.py 2>&1 | grep -E "host-buffer search|timeline" | sed -n '1p;12p'; done
echo "NO_OVERLAP"; DADE_GPU_NO_OVERLAP=1 DADE_GPU_TIMELINE=1 python tools/e2e_breakdown.py 2>&1 | grep -E "host-buffer search|timeline" | sed -n '1p;12p'
