#!/bin/bash
# rebuild the product library and the DIAG (phase profile / watchdog) variant
cd "$(dirname "$0")/.." && python -m paper_1705_09366_b200.build | tail -1 && python scripts/build_variant.py prof -DSTKDE_TC_DIAG=1 | tail -1
