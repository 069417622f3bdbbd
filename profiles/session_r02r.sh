#!/bin/bash
for f in 0 1; do for c in 0 1; do for t in 0 1; do timeout 120 python profiles/m2_factors.py $f $c $t 2>&1 | grep median; done; done; done
