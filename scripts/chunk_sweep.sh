#!/usr/bin/env bash
# Chunk-grid knob sweep for adr_paged_decode_attn (GPU box): each line is one
# process with the knobs in its environment (they are read once per process).
# ADR_SPLIT_RULE: 0 no sqrt rule, 1 sqrt rule, 2 (+ round up to 2^k), 3 (+ round down).
set -u
KNOBS=${KNOBS:-"default ADR_SPLIT_RULE=2 ADR_SPLIT_RULE=3 ADR_CHUNK_MIN=32 ADR_CHUNK_MIN=64"}
for knobs in $KNOBS; do
  echo "== knobs: ${knobs}"
  [ "$knobs" = default ] && knobs=""
  env ${knobs//,/ } timeout 300 python scripts/library_compare.py --only none --layers 6 --reps 10 \
      --configs ${CONFIGS:-C2,C3,C5} /tmp/cs.json 2>/dev/null | grep -E "ours \(adr"
done
