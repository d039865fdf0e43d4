// Host-only check of the prep kernel's CTA plans (prep.cuh: prep_map / prep_ctas, prep_map_ov / prep_ctas_ov) and of
// the UP raster-group rule (union.cuh: union_group_up): every (block, part) pair is produced exactly once, a block's
// parts have consecutive logical ids and agree on the part count, the count is a power of two dividing the block rows,
// and the window-position-major order puts every window's densest block first.  Runs on the CPU (no device code is
// executed); built and run by tests/test_prep_plan.py.
#include <cstdio>
#include <vector>
#include "../paper_2603_23198_b200/csrc/prep.cuh"

using namespace sffn;

static int fails = 0;
#define CHECK(c, ...)                         \
    do {                                      \
        if (!(c)) {                           \
            if (fails++ < 20) printf(__VA_ARGS__); \
        }                                     \
    } while (0)

static void check_plan(int NB, int WB, int base, int boost, bool ov, int tail_w0, int tail_split) {
    const int n = ov ? prep_ctas_ov(NB, WB, base, boost, tail_w0, tail_split) : prep_ctas(NB, WB, base, boost);
    std::vector<int> seen(static_cast<size_t>(NB) * 8, 0), parts(NB, 0), first(NB, -1), last(NB, -1);
    int prev_b = -1;
    for (int lid = 0; lid < n; ++lid) {
        int b, part;
        const int sp = ov ? prep_map_ov(lid, NB, WB, base, boost, tail_w0, tail_split, &b, &part)
                          : prep_map(lid, NB, WB, base, boost, &b, &part);
        CHECK(sp > 0 && b >= 0 && b < NB && part >= 0 && part < sp, "NB %d lid %d: b %d part %d sp %d\n", NB, lid, b, part, sp);
        if (!(sp > 0 && b >= 0 && b < NB)) continue;
        CHECK(sp <= META_SPLIT_MAX && (sp & (sp - 1)) == 0 && 128 % sp == 0, "bad part count %d\n", sp);
        CHECK(parts[b] == 0 || parts[b] == sp, "block %d: part counts %d vs %d\n", b, parts[b], sp);
        parts[b] = sp;
        seen[static_cast<size_t>(b) * 8 + part]++;
        if (b != prev_b) {
            CHECK(first[b] < 0, "block %d: parts not consecutive (lid %d)\n", b, lid);
            first[b] = lid;
        }
        last[b] = lid;
        prev_b = b;
    }
    int b_, p_;
    CHECK((ov ? prep_map_ov(n, NB, WB, base, boost, tail_w0, tail_split, &b_, &p_) : prep_map(n, NB, WB, base, boost, &b_, &p_)) == 0,
          "NB %d: id %d past the plan still maps\n", NB, n);
    for (int b = 0; b < NB; ++b) {
        CHECK(parts[b] > 0, "NB %d: block %d never planned\n", NB, b);
        for (int p = 0; p < parts[b]; ++p) CHECK(seen[static_cast<size_t>(b) * 8 + p] == 1, "block %d part %d seen %d\n", b, p, seen[b * 8 + p]);
        CHECK(last[b] - first[b] + 1 == parts[b], "block %d: ids %d..%d for %d parts\n", b, first[b], last[b], parts[b]);
    }
    if (!ov)  // position-major: every window's densest block (position 0) starts before any position-1 block
        for (int b = 0; b < NB; ++b)
            if (b % WB == 0)
                for (int c = 0; c < NB; ++c)
                    if (c % WB == 1) CHECK(first[b] < first[c], "NB %d: block %d after block %d\n", NB, b, c);
    if (ov && NB <= 260)  // window-major: every block of window w starts before any block of window w + 1
        for (int b = 0; b < NB; ++b)
            for (int c = 0; c < NB; ++c)
                if (b / WB < c / WB) CHECK(first[b] < first[c], "NB %d ov: block %d after block %d\n", NB, b, c);
}

int main() {
    for (int NB : {1, 2, 3, 15, 16, 17, 31, 32, 40, 128, 129, 256, 257, 512})
        for (int WB : {8, 16})
            for (int base : {1, 2, 4, 8})
                for (int boost : {0, 1, 2}) {
                    check_plan(NB, WB, base, boost, false, 0, 0);
                    const int nwin = (NB + WB - 1) / WB;
                    for (int tw0 : {0, nwin - 1, nwin}) check_plan(NB, WB, base, boost, true, tw0, 8 > base ? 8 : base);
                }
    // UP raster group: [8, 32], min(NB / 8, blocks whose X rows fill 32 MB)
    CHECK(union_group_up(256, 4096) == 32, "7B group %d\n", union_group_up(256, 4096));
    CHECK(union_group_up(512, 8192) == 16, "70B group %d\n", union_group_up(512, 8192));
    CHECK(union_group_up(128, 2048) == 16, "1B group %d\n", union_group_up(128, 2048));
    CHECK(union_group_up(32, 4096) == 8, "chunk group %d\n", union_group_up(32, 4096));
    for (int64_t NB = 1; NB < 4096; NB = NB * 3 + 1)
        for (int64_t K : {64, 256, 4096, 8192, 65536}) {
            const int g = union_group_up(NB, K);
            CHECK(g >= 8 && g <= 32 && g <= UNION_GROUP_MAX, "group %d\n", g);
        }
    printf(fails ? "FAIL %d\n" : "OK\n", fails);
    return fails ? 1 : 0;
}
