#!/bin/bash
# Same-box A/B of two libmgb builds on one command: tools/ab.sh LIB_A LIB_B REPS -- cmd...
# (alternates A, B, A, B ... so clock / power drift hits both)
A=$1; B=$2; N=$3; shift 4
for i in $(seq 1 $N); do
  echo "A: $(MGB_LIB=$A "$@" 2>&1 | tail -1 | cut -c1-200)"
  echo "B: $(MGB_LIB=$B "$@" 2>&1 | tail -1 | cut -c1-200)"
done
