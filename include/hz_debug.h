/* libhz test hooks — not part of the north-star ABI (include/hz.h).  Pure host logic, no GPU needed.
 *
 * hz_debug_plan_tiles: the work list of the complex64 tensor-map apply (apply27_tm) for one
 * slab of nx × ny × nz points (z0 = 0, nz_global = nz) whose PML-free index ranges are [lo_a, hi_a] per
 * axis (hi < lo: the whole axis is PML; lo = 0, hi = n-1: no PML), with `slots` resident CTAs on the GPU
 * and `nrhs` right-hand sides.  Writes up to max_items records of 5 ints {x0, y0, z0, z1, mode} to `out`
 * (caller-owned, 5*max_items ints; may be NULL when max_items = 0): the item's tile computes
 * [x0, x0+tx) × [y0, y0+ty) for local planes [z0, z1); mode 2 = x/y-PML body, 1 = z-PML body, 0 = PML-free
 * body.  tile_wh (may be NULL) receives {tx, ty}.  Returns the number of items (all of them, even when
 * more than max_items), or -1 on bad arguments.
 */
#ifndef HZ_DEBUG_H
#define HZ_DEBUG_H
#ifdef __cplusplus
extern "C" {
#endif

int hz_debug_plan_tiles(int nx, int ny, int nz, int lo_x, int hi_x, int lo_y, int hi_y, int lo_z, int hi_z, int slots,
                        int nrhs, int* out, int max_items, int* tile_wh);

#ifdef __cplusplus
}
#endif
#endif
