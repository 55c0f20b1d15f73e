// Tile geometry of the 5 x 10 tile join (join5.cu): how a node's nn new and no
// old candidates are laid out in slots and cut into tiles aligned to the
// reference's 5-blocking (compute_step, reference descent.hpp:82-153; block_core
// / tri_core5 and the flexible remainder paths, distance.hpp:134-190).  Host and
// device: tests/test_join5_geometry.py enumerates every (nn, no) through
// knng_cuda_debug_join5_pairs and checks that each pair of the node is evaluated
// exactly once, in the reference's fused / unfused class.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define KNNG_HD __host__ __device__ __forceinline__
#else
#define KNNG_HD inline
#endif

namespace knng_cuda {
namespace t5 {

// tile descriptor: node-relative slots
//   [0,7) ra   first row slot        [7,14) ca   first slot of column block A
//   [14,21) cb first slot of column block B      [21] column block B present
//   [22,24) kind (0 F, 1 U, 2 T, 3 dead)  [24,28) node index in the batch
//   [28] last tile of its pass group
constexpr uint32_t kKindF = 0, kKindU = 1, kKindT = 2;
KNNG_HD bool tile_dead(uint32_t tile) { return ((tile >> 22) & 3u) == 3u; }
constexpr uint32_t kThinCols = 24;  // T tile: 2 rows x 24 columns
KNNG_HD uint32_t make_tile(uint32_t v, uint32_t kind, uint32_t ra, uint32_t ca,
                                              uint32_t cb, bool has_b) {
    return ra | (ca << 7) | ((cb & 127u) << 14) | (uint32_t(has_b) << 21) | (kind << 22) |
           (v << 24);
}

struct Geom5 {
    uint32_t nn, no, fn, fo, m;
    uint32_t ro;    // leftover old candidates (slots [nn, nn + ro))
    uint32_t lrow;  // live leftover rows: slots [fn, fn + lrow)
    uint32_t ext;   // columns the first leftover row block runs against: [0, ext)
    bool thin_ok;   // thin tiles allowed (compile-time per kernel instantiation)
    KNNG_HD void set(uint32_t nn_, uint32_t no_, bool thin_ok_) {
        thin_ok = thin_ok_;
        nn = nn_;
        no = no_;
        fn = nn - nn % 5;
        ro = no % 5;
        fo = no - ro;
        m = nn + no;
        // leftover old candidates are rows only against fused new columns
        lrow = (nn - fn) + (fn ? ro : 0u);
        ext = nn > fn ? m : fn;
    }
    // slot -> position in the node's candidate order (new list, then old list)
    KNNG_HD uint32_t cand(uint32_t slot) const {
        if (slot < nn) return slot;
        const uint32_t x = slot - nn;
        return x < ro ? nn + fo + x : nn + x - ro;
    }
    KNNG_HD bool thin() const { return thin_ok && lrow <= 2; }
    KNNG_HD uint32_t f_tiles() const {
        const uint32_t nfb = fn / 5, nob = fo / 5;
        uint32_t t = 0;
        for (uint32_t i = 0; i < nfb; ++i) t += (nfb - i + nob + 1) / 2;
        return t;
    }
    KNNG_HD uint32_t u_tiles() const {
        if (!lrow || thin()) return 0u;
        return (ext + 9) / 10 + (lrow > 5 ? (fn + 9) / 10 : 0u);
    }
    KNNG_HD uint32_t t_tiles() const {
        return lrow && thin() ? (ext + kThinCols - 1) / kThinCols : 0u;
    }
    // t-th fused tile
    KNNG_HD uint32_t f_tile(uint32_t v, uint32_t t) const {
        const uint32_t nfb = fn / 5, nob = fo / 5;
        uint32_t i = 0;
        while (t >= (nfb - i + nob + 1) / 2) {
            t -= (nfb - i + nob + 1) / 2;
            ++i;
        }
        const uint32_t len = nfb - i + nob, q0 = 2 * t, q1 = 2 * t + 1;
        auto col = [&](uint32_t q) {
            return q < nfb - i ? 5 * (i + q) : nn + ro + 5 * (q - (nfb - i));
        };
        return make_tile(v, kKindF, 5 * i, col(q0), q1 < len ? col(q1) : 0u, q1 < len);
    }
    // t-th 5 x 10 leftover-row tile: the first row block over [0, ext), then
    // the second (leftover old rows only) over the fused new columns
    KNNG_HD uint32_t u_tile(uint32_t v, uint32_t t) const {
        const uint32_t na = (ext + 9) / 10;
        if (t < na) return make_tile(v, kKindU, fn, 10 * t, 10 * t + 5, 10 * t + 5 < ext);
        t -= na;
        return make_tile(v, kKindU, fn + 5, 10 * t, 10 * t + 5, 10 * t + 5 < fn);
    }
    // t-th thin tile
    KNNG_HD uint32_t t_tile(uint32_t v, uint32_t t) const {
        return make_tile(v, kKindT, fn, kThinCols * t, 0u, false);
    }
    // columns a leftover-row tile with first row ra runs against
    KNNG_HD uint32_t col_end(uint32_t ra) const { return ra == fn ? ext : fn; }
    // is (row slot r, column slot cc) a pair of the leftover-row tiles?  Every
    // unfused pair exactly once.
    KNNG_HD bool leftover_pair(uint32_t r, uint32_t cc) const {
        if (r < nn) return cc < m && (cc < fn || cc >= nn || cc > r);  // r >= fn: a leftover new row
        return r < fn + lrow && cc < fn;  // a leftover old row: fused new columns only
    }
    // Slot p (< 50) of a tile's accumulators: its (row slot, column slot), or
    // false when the slot is padding or the pair is not this tile's to count.
    // Every pair of the node comes out of exactly one slot of one tile, in the
    // reference's class: fused rows (r < fn) against new blocks j >= i or full
    // old blocks (F tiles), everything with a leftover row or column unfused.
    KNNG_HD bool tile_pair(uint32_t tile, uint32_t p, uint32_t& r, uint32_t& cc) const {
        const uint32_t kind = (tile >> 22) & 3u, ra = tile & 127u, ca = (tile >> 7) & 127u;
        const bool has_b = (tile >> 21) & 1u;
        if (kind == kKindT) {
            const uint32_t x = p / kThinCols, y = p % kThinCols;
            if (x >= 2) return false;
            r = ra + x;
            cc = ca + y;
        } else {
            const uint32_t x = p / 10u, y = p % 10u;
            if (x >= 5 || (y >= 5 && !has_b)) return false;
            r = ra + x;
            cc = y < 5 ? ca + y : ((tile >> 14) & 127u) + (y - 5);
        }
        return kind == kKindF ? (cc >= nn || cc > r) : leftover_pair(r, cc);
    }
};



}  // namespace t5
}  // namespace knng_cuda
