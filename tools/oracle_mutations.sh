#!/bin/bash
# Mutation check of the oracle pins: each plausible mistake below is applied to a
# scratch copy of oracle/mhfd_oracle.c and the -m "not gpu" pin suite must fail.
# Usage: tools/oracle_mutations.sh   (CPU only; a few minutes)
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
muts=(
 's/Di\[p\] = t\[i - 1\] \* (Lcur\[p\] - Lprev\[p\])/Di[p] = t[i] * (Lcur[p] - Lprev[p])/'            # wrong DoG scale index
 's/if (d > best) { best = d; bi = i; }/if (d >= best) { best = d; bi = i; }/'                          # last argmax on ties
 's/for (int d = -R; d <= R; ++d) w\[d + R\] \/= s;/;/'                                                 # dropped renormalisation
 's/acc += w\[b + R\] \* src\[wrap((int64_t)x + b, W)\]/acc += w[b + R] * src[wrap((int64_t)x - 2*b, W)]/'  # wrong tap index
 's/int64_t klo = (int64_t)floor(sat_low \* (double)npx);/int64_t klo = (int64_t)ceil(sat_low * (double)npx);/'  # rank rounding
 's/if (p->y != q->y) return p->y < q->y ? -1 : 1;/if (p->x != q->x) return p->x < q->x ? -1 : 1;/'      # transposed priority
 's/double rb = sqrt(2.0) \* t\[b->scale\];/double rb = sqrt(2.0) * t[b->scale + 1];/'                   # off-by-one radius
 's/if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue; \/\* -inf padding \*\//yy = (yy + H) % H; xx = (xx + W) % W;/'  # periodic NMS
 's/if (!(c > tau)) continue;/if (!(c >= tau)) continue;/'                                              # non-strict threshold
 's/const int64_t cell = (int64_t)ceil(2.0 \* rmax) + 1;/const int64_t cell = (int64_t)ceil(rmax);/'     # grid prune: cells < 2 r_max
 's/for (int64_t xx = cx - 1; xx <= cx + 1 \&\& ok; ++xx)/for (int64_t xx = cx; xx <= cx + 1 \&\& ok; ++xx)/'  # grid prune: missed cells
)
fail=0
for m in "${muts[@]}"; do
  rm -rf "$TMP/w" && mkdir "$TMP/w" && cp -r "$ROOT/oracle" "$ROOT/synth" "$ROOT/tests" "$ROOT/pytest.ini" "$TMP/w/"
  rm -f "$TMP"/w/oracle/*.so
  sed -i "$m" "$TMP/w/oracle/mhfd_oracle.c"
  if cmp -s "$ROOT/oracle/mhfd_oracle.c" "$TMP/w/oracle/mhfd_oracle.c"; then echo "NOT APPLIED: $m"; fail=1; continue; fi
  out=$(cd "$TMP/w" && timeout 600 python -m pytest tests/test_oracle_pins.py -q -x 2>&1 | tail -1)
  case "$out" in *failed*) echo "killed:   $m";; *) echo "SURVIVED: $m -> $out"; fail=1;; esac
done
rm -rf "$TMP"
exit $fail
