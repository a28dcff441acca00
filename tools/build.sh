#!/usr/bin/env bash
# Build the product library (libcct.so) and the CPU checker (oracle/).
set -euo pipefail
ROOT="$(cd "$(dirname "${BASH_SOURCE[0]}")/.." && pwd)"
make -s -C "$ROOT/paper_1504_04343_b200/csrc" -j"$(nproc)"
make -s -C "$ROOT/oracle"
