#!/bin/bash
# Round-2 BASELINE-size fixtures from the unmodified reference (CPU only, this
# container; hours of single-core work).  Jobs are paired so host RAM (62 GB)
# is never exceeded: C5's reference solve peaks near 50 GB and runs alone.
set -x
cd "$(dirname "$0")/.."
G="python oracle/make_golden.py"
$G curg:c1
$G capped200:c3 & $G capped200:c4 & wait
$G capped200:c5
$G cappedulp200:c3 & $G cappedulp200:c4 & wait
$G cappedulp200:c5
$G curg:c3
$G curg:c4
