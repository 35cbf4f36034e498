#!/bin/sh
# Golden for tests/test_cpp_dropin.py: tests/cpp/dropin_main.cpp compiled against
# the UNMODIFIED reference headers (/root/reference/proj/include) and linked with
# the reference library compiled from its own sources (oracle/_ref/libcmgref.so,
# oracle/Makefile), run once. Needs /root/reference (dev container only).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
make -s -C "$ROOT/oracle" ref
g++ -std=c++20 -O2 -I/root/reference/proj/include "$ROOT/tests/cpp/dropin_main.cpp" \
    "$ROOT/oracle/_ref/libcmgref.so" -Wl,-rpath,"$ROOT/oracle/_ref" -lpthread -o /tmp/cmgb_dropin_ref
/tmp/cmgb_dropin_ref > "$HERE/dropin_ref.json"
echo "wrote $HERE/dropin_ref.json"
for sc in box_on_plane capsule_vs_hollow; do
  /tmp/cmgb_dropin_ref "$ROOT/tests/scenes/$sc.json" "$HERE/dropin_${sc}_ref.csv" "$HERE/dropin_${sc}_ref.json"
done
# the reference's own dev probe (proj/tests/probe.cpp) on the reference build
g++ -std=c++20 -O2 -I/root/reference/proj/include /root/reference/proj/tests/probe.cpp \
    "$ROOT/oracle/_ref/libcmgref.so" -Wl,-rpath,"$ROOT/oracle/_ref" -lpthread -o /tmp/cmgb_probe_ref
/tmp/cmgb_probe_ref > "$HERE/probe_ref.txt"
/tmp/cmgb_probe_ref 0.06 0.0 0.0 0.01 0.005 0.02 5 0.05 -0.03 > "$HERE/probe_ref_tilt.txt"
echo "wrote $HERE/probe_ref.txt $HERE/probe_ref_tilt.txt"
