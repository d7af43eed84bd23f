#!/usr/bin/env bash
# TEST INFRASTRUCTURE: plants plausible mistakes in oracle.c one at a time and
# checks that tests/test_oracle_pins.py catches each (every line must report
# failures).  Restores oracle.c afterwards.
set -u
cd "$(dirname "$0")/.."
cp oracle/oracle.c /tmp/oracle.c.mut.bak
trap 'cp /tmp/oracle.c.mut.bak oracle/oracle.c; python -c "import oracle.oracle as o; o.build_lib(True)"' EXIT
for m in \
 's/return part\[u\] == part\[v\] ? 0 : w;/return w;/' \
 's/if (kind\[p\] == OR_KIND_RESIDUAL \&\& part\[p\] == h) continue;/;/' \
 's/if (nxt < 0 || s < nxt) nxt = s;/if (nxt < 0 || s > nxt) nxt = s;/' \
 's/int64_t len = tl\[p\] + c\[p\] + comm_eff/int64_t len = tl[p] + comm_eff/' \
 's/if (first_over\[q\] < 0 \&\& cur\[q\] > cap_eff\[q\])/if (first_over[q] < 0 \&\& cur[q] >= cap_eff[q])/' \
 's/if (kind\[n\] == OR_KIND_NORMAL) cur\[h\] += effmem\[n\];/;/' \
 's/bl\[u\] = c\[u\] + best;/bl[u] = best;/' \
 's/if (pos\[u\] > \*l) \*l = pos\[u\];/if (pos[u] < *l || *l < 0) *l = pos[u];/' \
 's/if (part\[u\] != part\[g->succ\[a\]\]) cut +=/if (part[u] == part[g->succ[a]]) cut +=/' \
 's/r->cp_end = r->cp_len ? cp\[r->cp_len - 1\] : -1;/r->cp_end = r->cp_len ? cp[0] : -1;/' \
 's/r->overflow_mask |= 1 << q;/r->overflow_mask |= 1 << (q + 1);/' \
 's/r->peak_pos\[q\] = in ? ppos\[q\] : -1;/r->peak_pos[q] = in ? ppos[q] : 0;/' \
 's/r->cp_start = r->cp_len ? cp\[0\] : -1;/r->cp_start = r->cp_len ? cp[1 % r->cp_len] : -1;/' \
 's/int64_t arrive = ft\[v\] + (part\[s\] == q ? 0 : w\[g->succ_eid\[a\]\]);/int64_t arrive = ft[v];/' \
 's/    if (a->level != b->level) return a->level < b->level;/    ;/' \
 's/st\[v\] = e.ready > free_at\[q\] ? e.ready : free_at\[q\];/st[v] = e.ready;/' \
 's/        free_at\[q\] = ft\[v\];/        ;/' \
 's/    if (a->ready != b->ready) return a->ready < b->ready;/    if (a->ready != b->ready) return a->ready > b->ready;/' \
 's/int64_t arrive = ft\[v\] + (part\[s\] == q ? 0 :/int64_t arrive = st[v] + (part[s] == q ? 0 :/' \
 's/(tl\[s\] + bl\[s\] == tl\[best\] + bl\[best\] \&\& s < best)/(tl[s] + bl[s] == tl[best] + bl[best] \&\& s > best)/' \
 's/                    if (cluster_of\[p\] >= 0) continue;/                    continue;/' \
 's/    if (x->w != y->w) return x->w > y->w ? -1 : 1;/    if (x->w != y->w) return x->w < y->w ? -1 : 1;/' \
 's/int rc = or_weighted_levels(g, c, w, cluster_of, tl, bl);/int rc = or_weighted_levels(g, c, w, NULL, tl, bl);/' \
 's/if (tl\[v\] + bl\[v\] > crit\[cluster_of\[v\]\])/if (tl[v] + bl[v] < crit[cluster_of[v]])/' \
 's/if (m + a\[pick\] <= cap_eff\[k\] \&\& (tgt < 0 || m < mcons/if (m + a[pick] <= cap_eff[k] \&\& (tgt < 0 || m > mcons/' \
 's/if (fo\[k\] >= 0 \&\& (q < 0 || fo\[k\] < fo\[q\])) q = k;/if (fo[k] >= 0 \&\& (q < 0 || fo[k] > fo[q])) q = k;/' \
 's/if (last >= 0 \&\& pos\[last\] >= i) a\[last\] += mem\[p\];/if (last >= 0 \&\& pos[last] > i) a[last] += mem[p];/' \
 's/if (part\[g->succ\[e\]\] == q) cost\[v\] += w\[g->succ_eid\[e\]\];/;/' \
 's/const int32_t pick = (B >= 0 \&\& cost\[B\] < cost\[A\]) ? B : A;/const int32_t pick = A;/' \
 's/const int cc = comm\[t\] > wsc \&\& comm\[t\] > work\[t\] \&\& comm\[t\] > U;/const int cc = 0;/' \
 's/    const int high_ccr = sum_w >= 10 \* sum_c;/    const int high_ccr = 0;/' \
 's/if (tgt < 0 || cost < best || (cost == best \&\& comm\[q\] > comm\[tgt\]))/if (tgt < 0 || cost < best)/' \
 's/if (cluster_of\[g->succ\[a\]\] != k \&\& g->level\[g->succ\[a\]\] - 1 < hi) hi = g->level\[g->succ\[a\]\] - 1;/if (cluster_of[g->succ[a]] != k \&\& g->level[g->succ[a]] < hi) hi = g->level[g->succ[a]];/' \
 's/const int64_t U = fw_range(unm, lo, hi) - wsc;/const int64_t U = fw_range(unm, lo, hi);/' \
 's/for (int32_t q = 1; q < K; ++q) if (comm\[q\] > comm\[t\]) t = q;/for (int32_t q = 1; q < K; ++q) if (comm[q] >= comm[t]) t = q;/' \
 's/            if (gain <= 0) continue;/            if (gain < 0) continue;/' \
 's/            if (mn > mb) continue;/            ;/' \
 's/if (best < 0 || gain > best_gain) { best = B; best_gain = gain; }/if (best < 0 || gain >= best_gain) { best = B; best_gain = gain; }/' \
 's/if (B == A || marked\[B\] || part\[hB\] == pa) continue;/if (B == A || part[hB] == pa) continue;/' \
 's/for (int32_t bi = lo; bi < ns \&\& seen < window; ++bi) {/for (int32_t bi = lo; bi < ns; ++bi) {/' \
 's/            if (bt < 0 || bL >= L_cur) break;/            if (bt < 0 || bL > L_cur) break;/' \
 's/if ((side == 0 \&\& k == 0) || (side == 1 \&\& k == cl - 1)) continue;/if ((side == 0 \&\& k == 0) || side == 1) continue;/' \
 's/if (rf_level_work(tree + (size_t)q \* (D + 1), D, l, l) + c\[n\] > mx) continue;/;/' \
 ; do
  cp /tmp/oracle.c.mut.bak oracle/oracle.c
  sed -i "$m" oracle/oracle.c
  r=$(timeout 300 python -m pytest tests/test_oracle_pins.py -q -p no:cacheprovider 2>&1 | tail -1)
  echo "$m => $r"
done
