/* libhz test hooks — not part of the north-star ABI (include/hz.h).  Pure host logic, no GPU needed.
 *
 * hz_debug_plan_tiles: the x/y tiles the complex64 apply (apply27_cp) uses for an nx × ny
 * plane whose PML-free index ranges are [lo_x, hi_x] and [lo_y, hi_y] (hi < lo: the whole axis is PML;
 * lo = 0, hi = n-1: no PML), with rows_per_thread = 1 or 2 (1: two RHS per CTA, 2: one RHS).
 * Writes up to max_tiles records of 9 ints {x0, y0, tx, ty, xs, ys, xe, ye, pml} to `out` (caller-owned,
 * 9*max_tiles ints; may be NULL when max_tiles = 0): the tile computes [x0, x0+tx) × [y0, y0+ty), stores
 * [xs, xe) × [ys, ye), pml = 1 if it runs the x/y-PML body.  Returns the number of tiles (all of them,
 * even when more than max_tiles), or -1 on bad arguments.
 */
#ifndef HZ_DEBUG_H
#define HZ_DEBUG_H
#ifdef __cplusplus
extern "C" {
#endif

int hz_debug_plan_tiles(int nx, int ny, int lo_x, int hi_x, int lo_y, int hi_y, int rows_per_thread, int* out,
                        int max_tiles);

#ifdef __cplusplus
}
#endif
#endif
