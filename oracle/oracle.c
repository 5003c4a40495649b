/*
 * CPU ORACLE — test infrastructure only, never the product path.
 *
 * A plain-C restatement of the reference `freeview` hot path
 * (/root/reference/pkg/src/freeview/<module>.py), float64 throughout, written to
 * reproduce the reference's IEEE-754 operation order bit for bit:
 *   - compiled with -ffp-contract=off, so every `a*b + c` rounds twice
 *     exactly like numpy's unfused ufuncs;
 *   - the one place the reference goes through BLAS (`pts @ R.T`,
 *     camera.py:177; `pc @ R`, camera.py:218) uses explicit fma() in the
 *     order OpenBLAS 0.3.30 evaluates it (pinned by
 *     tests/test_oracle_golden.py against reference outputs generated with
 *     OPENBLAS_CORETYPE=Haswell by scripts/make_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library, and only as the checker / the timed CPU baseline.
 *
 * Pinned: tests/golden/ holds outputs of the reference itself
 * (scripts/make_golden.py); tests/test_oracle_golden.py checks this file
 * against them on every CPU test run.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "mc_cases.h"

/* hot loops get an FMA-ISA clone when the host CPU has one (the result is
 * identical: fma() is exact either way, the clone only avoids a libm call) */
#define OR_HOT __attribute__((target_clones("arch=x86-64-v3", "default")))

/* Camera record; byte layout identical to `fvv_camera` in include/fvv.h. */
typedef struct {
    double R[9];
    double t[3];
    double fx, fy, cx, cy, skew;
    double k1, k2, p1, p2, k3;
    int32_t width, height, id, has_distortion;
} or_cam;

/* hull.py:20 — carve processes voxels in chunks of 2^20; a chunk holding a
 * single voxel reaches `project` as a (1,3) array, which numpy sends to
 * BLAS gemv (different FMA order) instead of gemm. */
#define OR_CARVE_CHUNK (1LL << 20)
/* visibility.py:19 */
#define OR_NEAR_CLIP_MM 1.0
/* mesh.py:22 */
#define OR_DEGENERATE_AREA 1e-9

/* ---------------------------------------------------------------- camera */

/* camera.py:177 `pts @ cam.rotation.T + cam.translation`.
 * gemm (N>=2): fma(z,R2, fma(y,R1, x*R0)) + t
 * gemv (N==1): fma(z,R2, fma(x,R0, y*R1)) + t */
static inline void or_world_to_cam(const or_cam *c, double x, double y, double z,
                                   int gemv, double pc[3]) {
    for (int r = 0; r < 3; ++r) {
        const double *R = c->R + 3 * r;
        double acc = gemv ? fma(x, R[0], y * R[1]) : fma(y, R[1], x * R[0]);
        pc[r] = fma(z, R[2], acc) + c->t[r];
    }
}

/* camera.py:164-201 (project) with camera.py:154-161 (distort). */
static inline void or_project1(const or_cam *c, double x, double y, double z,
                               int use_dist, int gemv, double *u, double *v,
                               double *zc, int *inf) {
    double pc[3];
    or_world_to_cam(c, x, y, z, gemv, pc);
    double zz = pc[2];
    double sz = (zz != 0.0) ? zz : 1.0;
    double xn = pc[0] / sz;
    double yn = pc[1] / sz;
    double xd, yd;
    if (use_dist && c->has_distortion) {
        double r2 = xn * xn + yn * yn;
        double radial = 1.0 + r2 * (c->k1 + r2 * (c->k2 + r2 * c->k3));
        xd = xn * radial + 2.0 * c->p1 * xn * yn + c->p2 * (r2 + 2.0 * xn * xn);
        yd = yn * radial + c->p1 * (r2 + 2.0 * yn * yn) + 2.0 * c->p2 * xn * yn;
    } else {
        xd = xn;
        yd = yn;
    }
    double uu = c->fx * (xd + c->skew * yd) + c->cx;
    double vv = c->fy * yd + c->cy;
    double iu = rint(uu), iv = rint(vv); /* np.rint: half to even */
    *u = uu;
    *v = vv;
    *zc = zz;
    *inf = (zz > 0.0) && (iu >= 0.0) && (iu <= (double)(c->width - 1)) &&
           (iv >= 0.0) && (iv <= (double)(c->height - 1));
}

OR_HOT void or_project(const or_cam *c, const double *pts, int64_t n, int use_dist,
                double *px, double *z, uint8_t *inf) {
    int gemv = (n == 1);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        int in;
        or_project1(c, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], use_dist, gemv,
                    &px[2 * i], &px[2 * i + 1], &z[i], &in);
        inf[i] = (uint8_t)in;
    }
}

/* ---------------------------------------------------------------- voxels */

/* voxels.py:46-56: c = origin + spacing * (ijk + 0.5) */
static inline void or_center(const double *origin, double spacing, const int64_t *dims,
                             int64_t l, double c[3]) {
    int64_t nx = dims[0], ny = dims[1];
    int64_t i = l % nx, j = (l / nx) % ny, k = l / (nx * ny);
    c[0] = origin[0] + spacing * ((double)i + 0.5);
    c[1] = origin[1] + spacing * ((double)j + 0.5);
    c[2] = origin[2] + spacing * ((double)k + 0.5);
}

/* ------------------------------------------------------------------ hull */

/* hull.py:78-119 (_carve_chunk + carve). Silhouettes are uint8 0/1 masks in
 * rig order, camera c's (H, W) mask at sils + sil_off[c]. */
OR_HOT void or_carve(const or_cam *cams, int ncam, const uint8_t *sils, const int64_t *sil_off,
              const double *origin, double spacing, const int64_t *dims, int min_views,
              uint8_t *occ) {
    int64_t nvox = dims[0] * dims[1] * dims[2];
    int64_t gemv_voxel = (nvox % OR_CARVE_CHUNK == 1) ? nvox - 1 : -1;
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t l = 0; l < nvox; ++l) {
        double p[3];
        or_center(origin, spacing, dims, l, p);
        int gemv = (l == gemv_voxel);
        int seen = 0, keep = 1;
        for (int c = 0; c < ncam && keep; ++c) {
            double u, v, z;
            int in;
            or_project1(&cams[c], p[0], p[1], p[2], 1, gemv, &u, &v, &z, &in);
            if (!in) continue;
            ++seen;
            int64_t iu = (int64_t)rint(u), iv = (int64_t)rint(v);
            if (!sils[sil_off[c] + iv * cams[c].width + iu]) keep = 0;
        }
        occ[l] = (uint8_t)(keep && seen >= min_views);
    }
}

/* hull.py:218-254 semantics, by an independent algorithm: 26-neighbour BFS
 * seeded in ascending linear index, so label n is the component whose
 * minimum linear index is the n-th smallest (hull.py:195-197). Writes
 * labels (0 = background) and per component {count, bbmin[3], bbmax[3]}
 * (inclusive voxel indices, hull.py:201-214). Returns the component count. */
int64_t or_label(const uint8_t *occ, const int64_t *dims, int32_t *labels, int64_t *comps) {
    int64_t nx = dims[0], ny = dims[1], nz = dims[2];
    int64_t nvox = nx * ny * nz;
    memset(labels, 0, (size_t)nvox * sizeof(int32_t));
    int64_t n_on = 0;
    for (int64_t l = 0; l < nvox; ++l) n_on += occ[l] != 0;
    if (!n_on) return 0;
    int64_t *queue = (int64_t *)malloc((size_t)n_on * sizeof(int64_t));
    int64_t ncomp = 0;
    for (int64_t seed = 0; seed < nvox; ++seed) {
        if (!occ[seed] || labels[seed]) continue;
        int32_t lab = (int32_t)(++ncomp);
        int64_t *cs = comps + 7 * (ncomp - 1);
        cs[0] = 0;
        cs[1] = cs[2] = cs[3] = INT64_MAX;
        cs[4] = cs[5] = cs[6] = -1;
        int64_t head = 0, tail = 0;
        queue[tail++] = seed;
        labels[seed] = lab;
        while (head < tail) {
            int64_t l = queue[head++];
            int64_t i = l % nx, j = (l / nx) % ny, k = l / (nx * ny);
            cs[0] += 1;
            if (i < cs[1]) cs[1] = i;
            if (j < cs[2]) cs[2] = j;
            if (k < cs[3]) cs[3] = k;
            if (i > cs[4]) cs[4] = i;
            if (j > cs[5]) cs[5] = j;
            if (k > cs[6]) cs[6] = k;
            for (int dk = -1; dk <= 1; ++dk)
                for (int dj = -1; dj <= 1; ++dj)
                    for (int di = -1; di <= 1; ++di) {
                        int64_t ii = i + di, jj = j + dj, kk = k + dk;
                        if (ii < 0 || jj < 0 || kk < 0 || ii >= nx || jj >= ny || kk >= nz) continue;
                        int64_t m = ii + nx * (jj + ny * kk);
                        if (occ[m] && !labels[m]) {
                            labels[m] = lab;
                            queue[tail++] = m;
                        }
                    }
        }
    }
    free(queue);
    return ncomp;
}

/* ------------------------------------------------------------------ mesh */

/* mesh.py:25-38: Bourke cube corners and edge (base offset, axis). */
static const int OR_CORNER[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                    {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
static const int OR_EDGE_BASE[12][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 0},
                                        {0, 0, 1}, {1, 0, 1}, {0, 1, 1}, {0, 0, 1},
                                        {0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}};
static const int OR_EDGE_AXIS[12] = {0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2};

static inline int or_hexval(char ch) { return ch <= '9' ? ch - '0' : ch - 'a' + 10; }

typedef struct {
    int64_t nv, nt;
    double *verts;     /* (nv, 3) */
    int32_t *tris;     /* (nt, 3) */
    int64_t fallback_edges, inconsistent_starts;
} or_mesh;

void or_mesh_free(or_mesh *m) {
    free(m->verts);
    free(m->tris);
    m->verts = NULL;
    m->tris = NULL;
}

/* mesh.py:131-162 closed-form Bresenham pixel t of the segment a->b. */
static inline void or_bresenham_px(int64_t ax, int64_t ay, int64_t bx, int64_t by, int64_t t,
                                   int64_t *x, int64_t *y) {
    int64_t dx = llabs(bx - ax), dy = llabs(by - ay);
    int64_t sx = bx >= ax ? 1 : -1, sy = by >= ay ? 1 : -1;
    int64_t major = dx > dy ? dx : dy;
    int xmajor = dx >= dy;
    int64_t dmaj = major > 1 ? major : 1;
    int64_t dmin = xmajor ? dy : dx;
    int64_t tc = t < major ? t : major;
    int64_t smin = (2 * tc * dmin + dmaj) / (2 * dmaj); /* all operands >= 0 */
    *x = ax + sx * (xmajor ? tc : smin);
    *y = ay + sy * (xmajor ? smin : tc);
}

/* mesh.py:231-272 (_edge_isovalues_batch) for one edge; cameras visited in
 * ascending id order (order[]), strict `<` so ties keep the lowest id. */
static double or_edge_lambda(const or_cam *cams, const int *order, int ncam, const uint8_t *sils,
                             const int64_t *sil_off, const double *pon, const double *poff,
                             int gemv, int64_t *inconsistent, int *cam_sel) {
    double lam = INFINITY;
    int sel = -1;
    for (int oi = 0; oi < ncam; ++oi) {
        int c = order[oi];
        const or_cam *cam = &cams[c];
        double uo, vo, zo, uf, vf, zf;
        int ino, inf;
        or_project1(cam, pon[0], pon[1], pon[2], 1, gemv, &uo, &vo, &zo, &ino);
        or_project1(cam, poff[0], poff[1], poff[2], 1, gemv, &uf, &vf, &zf, &inf);
        if (!(ino && inf)) continue;
        int64_t ax = (int64_t)rint(uo), ay = (int64_t)rint(vo);
        int64_t bx = (int64_t)rint(uf), by = (int64_t)rint(vf);
        int64_t dx = llabs(bx - ax), dy = llabs(by - ay);
        int64_t len = (dx > dy ? dx : dy) + 1;
        const uint8_t *sil = sils + sil_off[c];
        int64_t W = cam->width;
        int64_t first_bg = -1;
        int64_t lx = 0, ly = 0;
        for (int64_t t = 0; t < len; ++t) {
            int64_t x, y;
            or_bresenham_px(ax, ay, bx, by, t, &x, &y);
            if (!sil[y * W + x]) {
                first_bg = t;
                break;
            }
        }
        int start_bg = (first_bg == 0);
        double ddx = uf - uo, ddy = vf - vo;
        double denom = sqrt(ddx * ddx + ddy * ddy);
        double lam_i = 1.0;
        if (start_bg) {
            *inconsistent += 1;
            lam_i = 0.0;
        } else if (first_bg > 0 && denom > 1e-12) {
            or_bresenham_px(ax, ay, bx, by, first_bg - 1, &lx, &ly);
            double ex = (double)lx - uo, ey = (double)ly - vo;
            double q = sqrt(ex * ex + ey * ey) / denom;
            lam_i = q < 0.0 ? 0.0 : (q > 1.0 ? 1.0 : q);
        }
        if (lam_i < lam) {
            lam = lam_i;
            sel = cam->id;
        }
    }
    *cam_sel = sel;
    return sel == -1 ? 0.5 : lam;
}

/* mesh.py:275-374 (polygonize). exact != 0: silhouette-exact isovalues,
 * else every vertex at fixed_iso. Returns 0, or -1 on allocation failure. */
OR_HOT int or_polygonize(const uint8_t *occ, const double *origin, double spacing, const int64_t *dims,
                  const or_cam *cams, int ncam, const uint8_t *sils, const int64_t *sil_off,
                  int exact, double fixed_iso, or_mesh *out) {
    memset(out, 0, sizeof(*out));
    int64_t nx = dims[0], ny = dims[1], nz = dims[2];
    if (nx < 2 || ny < 2 || nz < 2) return 0;
    int64_t nvox = nx * ny * nz;
#define VOL(i, j, k) (occ[(i) + nx * ((j) + ny * (k))] != 0)

    /* surface cells, C order over (nx-1, ny-1, nz-1) (mesh.py:302-306) */
    int64_t nsurf = 0;
    for (int64_t i = 0; i < nx - 1; ++i)
        for (int64_t j = 0; j < ny - 1; ++j)
            for (int64_t k = 0; k < nz - 1; ++k) {
                int ci = 0;
                for (int b = 0; b < 8; ++b)
                    ci |= VOL(i + OR_CORNER[b][0], j + OR_CORNER[b][1], k + OR_CORNER[b][2]) << b;
                nsurf += (ci > 0 && ci < 255);
            }
    if (!nsurf) return 0;

    /* intersected grid edges per axis, C order over the axis-shortened
     * shape (mesh.py:315-327); vmap: global edge id -> vertex index */
    int32_t *vmap = (int32_t *)malloc((size_t)(3 * nvox) * sizeof(int32_t));
    if (!vmap) return -1;
    int64_t ne = 0;
    for (int a = 0; a < 3; ++a) {
        int64_t ex = nx - (a == 0), ey = ny - (a == 1), ez = nz - (a == 2);
        for (int64_t i = 0; i < ex; ++i)
            for (int64_t j = 0; j < ey; ++j)
                for (int64_t k = 0; k < ez; ++k) {
                    int lo = VOL(i, j, k);
                    int hi = VOL(i + (a == 0), j + (a == 1), k + (a == 2));
                    int64_t gid = a * nvox + i + nx * (j + ny * k);
                    vmap[gid] = (lo != hi) ? (int32_t)ne++ : -1;
                }
        if (a < 2) {
            /* ids on the shortened face are never intersected */
        }
    }
    double *pon = (double *)malloc((size_t)ne * 3 * sizeof(double));
    double *poff = (double *)malloc((size_t)ne * 3 * sizeof(double));
    double *verts = (double *)malloc((size_t)(ne ? ne : 1) * 3 * sizeof(double));
    if (!pon || !poff || !verts) return -1;
    {
        int64_t e = 0;
        for (int a = 0; a < 3; ++a) {
            int64_t ex = nx - (a == 0), ey = ny - (a == 1), ez = nz - (a == 2);
            for (int64_t i = 0; i < ex; ++i)
                for (int64_t j = 0; j < ey; ++j)
                    for (int64_t k = 0; k < ez; ++k) {
                        int lo = VOL(i, j, k);
                        int hi = VOL(i + (a == 0), j + (a == 1), k + (a == 2));
                        if (lo == hi) continue;
                        double p0[3], p1[3];
                        int64_t b[3] = {i, j, k};
                        for (int d = 0; d < 3; ++d) {
                            p0[d] = origin[d] + spacing * ((double)b[d] + 0.5);
                            p1[d] = p0[d] + spacing * (double)(d == a);
                        }
                        for (int d = 0; d < 3; ++d) {
                            pon[3 * e + d] = lo ? p0[d] : p1[d];
                            poff[3 * e + d] = lo ? p1[d] : p0[d];
                        }
                        ++e;
                    }
        }
    }

    /* isovalues (mesh.py:332-336) and vertices (mesh.py:337) */
    int64_t inconsistent = 0, fallback = 0;
    int *order = (int *)malloc((size_t)(ncam > 0 ? ncam : 1) * sizeof(int));
    for (int c = 0; c < ncam; ++c) order[c] = c;
    for (int a = 1; a < ncam; ++a) /* sort positions by camera id (mesh.py:165-167) */
        for (int b = a; b > 0 && cams[order[b]].id < cams[order[b - 1]].id; --b) {
            int tmp = order[b];
            order[b] = order[b - 1];
            order[b - 1] = tmp;
        }
    int gemv = (ne == 1);
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : inconsistent, fallback)
    for (int64_t e = 0; e < ne; ++e) {
        double lam;
        if (exact) {
            int sel;
            lam = or_edge_lambda(cams, order, ncam, sils, sil_off, pon + 3 * e, poff + 3 * e, gemv,
                                 &inconsistent, &sel);
            fallback += (sel == -1);
        } else {
            lam = fixed_iso;
        }
        for (int d = 0; d < 3; ++d)
            verts[3 * e + d] = pon[3 * e + d] + lam * (poff[3 * e + d] - pon[3 * e + d]);
    }
    free(order);
    free(pon);
    free(poff);

    /* triangles: slot-major, then cell C order (mesh.py:351-359), winding
     * reversed (mesh.py:365), area > 1e-9 kept in order (mesh.py:372-373) */
    int32_t *tris = (int32_t *)malloc((size_t)nsurf * 5 * 3 * sizeof(int32_t));
    if (!tris) return -1;
    int64_t nt = 0;
    for (int slot = 0; slot < 5; ++slot) {
        for (int64_t i = 0; i < nx - 1; ++i)
            for (int64_t j = 0; j < ny - 1; ++j)
                for (int64_t k = 0; k < nz - 1; ++k) {
                    int ci = 0;
                    for (int b = 0; b < 8; ++b)
                        ci |= VOL(i + OR_CORNER[b][0], j + OR_CORNER[b][1], k + OR_CORNER[b][2]) << b;
                    if (ci == 0 || ci == 255) continue;
                    const char *cs = OR_MC_CASES[ci];
                    if ((int64_t)strlen(cs) < 3 * (slot + 1)) continue;
                    int32_t v[3];
                    for (int q = 0; q < 3; ++q) {
                        int e = or_hexval(cs[3 * slot + q]);
                        int64_t bi = i + OR_EDGE_BASE[e][0], bj = j + OR_EDGE_BASE[e][1],
                                bk = k + OR_EDGE_BASE[e][2];
                        v[q] = vmap[OR_EDGE_AXIS[e] * nvox + bi + nx * (bj + ny * bk)];
                    }
                    int32_t r0 = v[2], r1 = v[1], r2 = v[0];
                    const double *A = verts + 3 * r0, *B = verts + 3 * r1, *C = verts + 3 * r2;
                    double a0 = B[0] - A[0], a1 = B[1] - A[1], a2 = B[2] - A[2];
                    double b0 = C[0] - A[0], b1 = C[1] - A[1], b2 = C[2] - A[2];
                    double c0 = a1 * b2 - a2 * b1; /* numpy cross order (numeric.py) */
                    double c1 = a2 * b0 - a0 * b2;
                    double c2 = a0 * b1 - a1 * b0;
                    double area = 0.5 * sqrt((c0 * c0 + c1 * c1) + c2 * c2);
                    if (!(area > OR_DEGENERATE_AREA)) continue;
                    tris[3 * nt] = r0;
                    tris[3 * nt + 1] = r1;
                    tris[3 * nt + 2] = r2;
                    ++nt;
                }
    }
#undef VOL
    free(vmap);
    out->nv = ne;
    out->nt = nt;
    out->verts = verts;
    out->tris = tris;
    out->fallback_edges = exact ? fallback : 0;
    out->inconsistent_starts = exact ? inconsistent : 0;
    return 0;
}

/* ------------------------------------------------------------ visibility */

static inline int or_top_left(double ax, double ay, double bx, double by) {
    double dy = by - ay, dx = bx - ax; /* visibility.py:28-31 */
    return dy < 0.0 || (dy == 0.0 && dx < 0.0);
}

/* visibility.py:34-98 (rasterize). Rows [row0, row1) only, so callers can
 * split the image across threads without changing any pixel's result. */
static void or_raster_rows(const double *px, const double *pz, const int32_t *tris,
                           const int64_t *list, int64_t nlist, const or_cam *cam, double *depth,
                           int32_t *tri_id, int64_t row0, int64_t row1) {
    int64_t W = cam->width, H = cam->height;
    for (int64_t li = 0; li < nlist; ++li) {
        int64_t t = list[li];
        const int32_t *tv = tris + 3 * t;
        double x0 = px[2 * tv[0]], y0 = px[2 * tv[0] + 1];
        double x1 = px[2 * tv[1]], y1 = px[2 * tv[1] + 1];
        double x2 = px[2 * tv[2]], y2 = px[2 * tv[2] + 1];
        double za = pz[tv[0]], zb = pz[tv[1]], zc = pz[tv[2]];
        if (!(za > OR_NEAR_CLIP_MM && zb > OR_NEAR_CLIP_MM && zc > OR_NEAR_CLIP_MM)) continue;
        double mnx = fmin(fmin(x0, x1), x2), mxx = fmax(fmax(x0, x1), x2);
        double mny = fmin(fmin(y0, y1), y2), mxy = fmax(fmax(y0, y1), y2);
        if (isnan(x0) || isnan(x1) || isnan(x2) || isnan(y0) || isnan(y1) || isnan(y2)) continue;
        double flx = floor(mnx), fly = floor(mny), chx = ceil(mxx), chy = ceil(mxy);
        if (flx > (double)(W - 1) || fly > (double)(H - 1) || chx < 0.0 || chy < 0.0) continue;
        int64_t lox = flx > 0.0 ? (int64_t)flx : 0, loy = fly > 0.0 ? (int64_t)fly : 0;
        int64_t hix = chx < (double)(W - 1) ? (int64_t)chx : W - 1;
        int64_t hiy = chy < (double)(H - 1) ? (int64_t)chy : H - 1;
        if (hix < lox || hiy < loy) continue;
        double area = (x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0);
        if (area == 0.0) continue;
        if (area < 0.0) {
            double tx = x1, ty = y1;
            x1 = x2; y1 = y2; x2 = tx; y2 = ty;
            double tz = zb; zb = zc; zc = tz;
            area = -area;
        }
        int tl0 = or_top_left(x1, y1, x2, y2);
        int tl1 = or_top_left(x2, y2, x0, y0);
        int tl2 = or_top_left(x0, y0, x1, y1);
        int64_t ya = loy > row0 ? loy : row0, yb = hiy < row1 - 1 ? hiy : row1 - 1;
        for (int64_t y = ya; y <= yb; ++y) {
            double gy = (double)y;
            for (int64_t x = lox; x <= hix; ++x) {
                double gx = (double)x;
                double w0 = (x2 - x1) * (gy - y1) - (y2 - y1) * (gx - x1);
                double w1 = (x0 - x2) * (gy - y2) - (y0 - y2) * (gx - x2);
                double w2 = (x1 - x0) * (gy - y0) - (y1 - y0) * (gx - x0);
                int in = (w0 > 0.0 || (w0 == 0.0 && tl0)) && (w1 > 0.0 || (w1 == 0.0 && tl1)) &&
                         (w2 > 0.0 || (w2 == 0.0 && tl2));
                if (!in) continue;
                double b0 = w0 / area, b1 = w1 / area, b2 = w2 / area;
                double zinv = b0 / za + b1 / zb + b2 / zc;
                double d = 1.0 / zinv;
                int64_t p = y * W + x;
                if (d < depth[p]) {
                    depth[p] = d;
                    tri_id[p] = (int32_t)t;
                }
            }
        }
    }
}

OR_HOT void or_rasterize(const double *verts, int64_t nv, const int32_t *tris, int64_t nt,
                  const or_cam *cam, double *depth, int32_t *tri_id) {
    int64_t W = cam->width, H = cam->height;
    for (int64_t p = 0; p < W * H; ++p) {
        depth[p] = INFINITY;
        tri_id[p] = -1;
    }
    if (nt == 0) return;
    double *px = (double *)malloc((size_t)nv * 2 * sizeof(double));
    double *pz = (double *)malloc((size_t)nv * sizeof(double));
    int gemv = (nv == 1);
    for (int64_t i = 0; i < nv; ++i) {
        int in;
        or_project1(cam, verts[3 * i], verts[3 * i + 1], verts[3 * i + 2], 0, gemv, &px[2 * i],
                    &px[2 * i + 1], &pz[i], &in);
    }
    /* bin triangles into 16-row bands (ascending id inside each band), so
     * bands rasterise independently; a pixel's result only depends on the
     * triangles covering it, visited in ascending id exactly as before. */
    const int64_t band = 16, nband = (H + band - 1) / band;
    int64_t *cnt = (int64_t *)calloc((size_t)nband + 1, sizeof(int64_t));
    int64_t *b0 = (int64_t *)malloc((size_t)nt * sizeof(int64_t));
    int64_t *b1 = (int64_t *)malloc((size_t)nt * sizeof(int64_t));
    for (int64_t t = 0; t < nt; ++t) {
        const int32_t *tv = tris + 3 * t;
        double y0 = px[2 * tv[0] + 1], y1 = px[2 * tv[1] + 1], y2 = px[2 * tv[2] + 1];
        double mny = fmin(fmin(y0, y1), y2), mxy = fmax(fmax(y0, y1), y2);
        b0[t] = 1;
        b1[t] = 0; /* empty unless the row span meets the image */
        if (isnan(mny) || isnan(mxy)) continue;
        double fly = floor(mny), chy = ceil(mxy);
        if (fly > (double)(H - 1) || chy < 0.0) continue;
        int64_t lo = fly > 0.0 ? (int64_t)fly : 0;
        int64_t hi = chy < (double)(H - 1) ? (int64_t)chy : H - 1;
        b0[t] = lo / band;
        b1[t] = hi / band;
        for (int64_t b = b0[t]; b <= b1[t]; ++b) cnt[b + 1] += 1;
    }
    for (int64_t b = 0; b < nband; ++b) cnt[b + 1] += cnt[b];
    int64_t *lists = (int64_t *)malloc((size_t)(cnt[nband] > 0 ? cnt[nband] : 1) * sizeof(int64_t));
    int64_t *fill = (int64_t *)malloc((size_t)nband * sizeof(int64_t));
    for (int64_t b = 0; b < nband; ++b) fill[b] = cnt[b];
    for (int64_t t = 0; t < nt; ++t)
        for (int64_t b = b0[t]; b <= b1[t]; ++b) lists[fill[b]++] = t;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nband; ++b) {
        int64_t r0 = b * band;
        or_raster_rows(px, pz, tris, lists + cnt[b], cnt[b + 1] - cnt[b], cam, depth, tri_id, r0,
                       r0 + band < H ? r0 + band : H);
    }
    free(cnt);
    free(b0);
    free(b1);
    free(lists);
    free(fill);
    free(px);
    free(pz);
}

/* visibility.py:106-129 (classify_visibility); centroid = ((v0+v1)+v2)/3
 * (mesh.py:84-85, numpy mean). */
OR_HOT void or_classify(const double *verts, const int32_t *tris, int64_t nt, const or_cam *cam,
                 const double *depth, double t_v, uint8_t *vis) {
    int gemv = (nt == 1);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < nt; ++t) {
        const double *A = verts + 3 * tris[3 * t], *B = verts + 3 * tris[3 * t + 1],
                     *C = verts + 3 * tris[3 * t + 2];
        double c[3];
        for (int d = 0; d < 3; ++d) c[d] = ((A[d] + B[d]) + C[d]) / 3.0;
        double u, v, z;
        int in;
        or_project1(cam, c[0], c[1], c[2], 0, gemv, &u, &v, &z, &in);
        int visible = 0;
        if (in) {
            int64_t iu = (int64_t)rint(u), iv = (int64_t)rint(v);
            visible = (z - depth[iv * cam->width + iu]) <= t_v;
        }
        vis[t] = (uint8_t)visible;
    }
}

/* ---------------------------------------------------------------- render */

/* camera.py:204-220 (back_project, zero distortion) for one pixel.
 * `(pc - t) @ R`: gemm chain for >= 2 pixels; for a single pixel numpy
 * calls gemv, whose OpenBLAS Haswell kernel sums unfused. */
static inline void or_back_project(const or_cam *c, double pxu, double pxv, double d, int gemv,
                                   double pw[3]) {
    double yn = (pxv - c->cy) / c->fy;
    double xn = (pxu - c->cx) / c->fx - c->skew * yn;
    double q[3] = {xn * d - c->t[0], yn * d - c->t[1], d - c->t[2]};
    for (int col = 0; col < 3; ++col) {
        double r0 = c->R[col], r1 = c->R[3 + col], r2 = c->R[6 + col];
        pw[col] = gemv ? (q[0] * r0 + q[1] * r1) + q[2] * r2 : fma(q[2], r2, fma(q[1], r1, q[0] * r0));
    }
}

/* render.py:46-61 (sample_bilinear), one sample, 3 channels. */
static inline void or_bilinear(const uint8_t *img, int64_t W, int64_t H, double u, double v,
                               double out[3]) {
    u = fmin(fmax(u, 0.0), (double)W - 1.0);
    v = fmin(fmax(v, 0.0), (double)H - 1.0);
    int64_t x0 = (int64_t)floor(u), y0 = (int64_t)floor(v);
    int64_t x1 = x0 + 1 < W - 1 ? x0 + 1 : W - 1;
    int64_t y1 = y0 + 1 < H - 1 ? y0 + 1 : H - 1;
    double fx = u - (double)x0, fy = v - (double)y0;
    for (int ch = 0; ch < 3; ++ch) {
        double a = img[(y0 * W + x0) * 3 + ch], b = img[(y0 * W + x1) * 3 + ch];
        double c = img[(y1 * W + x0) * 3 + ch], d = img[(y1 * W + x1) * 3 + ch];
        double top = a * (1.0 - fx) + b * fx;
        double bot = c * (1.0 - fx) + d * fx;
        out[ch] = top * (1.0 - fy) + bot * fy;
    }
}

/* render.py:64-113 (render_view) given the per-triangle sources of
 * render.py:35-43 (computed by the caller from the ranking). Frames are
 * (H, W, 3) uint8 in rig order at frames + frame_off[c]. */
OR_HOT void or_render(const double *verts, int64_t nv, const int32_t *tris, int64_t nt,
               const int32_t *tri_src, const or_cam *rig, int ncam, const uint8_t *frames,
               const int64_t *frame_off, const or_cam *virt, const uint8_t *fallback,
               uint8_t *color, int32_t *source, uint8_t *covered) {
    int64_t W = virt->width, H = virt->height, np_ = W * H;
    double *depth = (double *)malloc((size_t)np_ * sizeof(double));
    int32_t *tid = (int32_t *)malloc((size_t)np_ * sizeof(int32_t));
    or_rasterize(verts, nv, tris, nt, virt, depth, tid);
    int64_t ncov = 0;
    for (int64_t p = 0; p < np_; ++p) {
        covered[p] = tid[p] >= 0;
        ncov += covered[p];
        source[p] = -1;
        color[3 * p] = color[3 * p + 1] = color[3 * p + 2] = 0;
    }
    /* pixels per source camera, for numpy's single-row gemv rule */
    int64_t *per_cam = (int64_t *)calloc((size_t)(ncam > 0 ? ncam : 1), sizeof(int64_t));
    int *pos_of = (int *)malloc((size_t)np_ * sizeof(int));
    for (int64_t p = 0; p < np_; ++p) {
        pos_of[p] = -1;
        if (!covered[p]) continue;
        int32_t s = tri_src[tid[p]];
        if (s < 0) continue;
        for (int c = 0; c < ncam; ++c)
            if (rig[c].id == s) {
                pos_of[p] = c;
                per_cam[c] += 1;
                break;
            }
    }
    int bp_gemv = (ncov == 1);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < np_; ++p) {
        if (!covered[p]) continue;
        int32_t s = tri_src[tid[p]];
        source[p] = s;
        if (s < 0) {
            for (int ch = 0; ch < 3; ++ch) color[3 * p + ch] = fallback[ch];
            continue;
        }
        int c = pos_of[p];
        double pw[3];
        or_back_project(virt, (double)(p % W), (double)(p / W), depth[p], bp_gemv, pw);
        double u, v, z;
        int in;
        or_project1(&rig[c], pw[0], pw[1], pw[2], 1, per_cam[c] == 1, &u, &v, &z, &in);
        double rgb[3];
        or_bilinear(frames + frame_off[c], rig[c].width, rig[c].height, u, v, rgb);
        for (int ch = 0; ch < 3; ++ch) {
            double q = rint(rgb[ch]);
            q = q < 0.0 ? 0.0 : (q > 255.0 ? 255.0 : q);
            color[3 * p + ch] = (uint8_t)q;
        }
    }
    free(per_cam);
    free(pos_of);
    free(depth);
    free(tid);
}

/* ------------------------------------------------------------ silhouette */

/* silhouette.py:59-69 distance_map: exact Euclidean distance to the nearest
 * proposal pixel (scipy.ndimage.distance_transform_edt(~prop)), computed as
 * sqrt of the exact integer squared distance. Independent algorithm from the
 * GPU kernels: per-column nearest feature, then per row the brute-force
 * minimum over candidate columns pruned by the running best. Returns 0, or 1
 * when the proposal is empty (caller fills +inf, silhouette.py:67-68). */
OR_HOT int or_distance_map(const uint8_t *prop, int64_t H, int64_t W, double *out) {
    int64_t nfg = 0;
    for (int64_t p = 0; p < H * W; ++p) nfg += prop[p] != 0;
    if (!nfg) return 1;
    const int64_t INF = (int64_t)1 << 40;
    int64_t *g = (int64_t *)malloc((size_t)(H * W) * sizeof(int64_t)); /* squared vertical */
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < W; ++x) {
        int64_t last = -1;
        for (int64_t y = 0; y < H; ++y) {
            if (prop[y * W + x]) last = y;
            g[y * W + x] = last < 0 ? INF : (y - last) * (y - last);
        }
        last = -1;
        for (int64_t y = H - 1; y >= 0; --y) {
            if (prop[y * W + x]) last = y;
            if (last >= 0) {
                int64_t d = (last - y) * (last - y);
                if (d < g[y * W + x]) g[y * W + x] = d;
            }
        }
    }
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t y = 0; y < H; ++y) {
        const int64_t *gr = g + y * W;
        for (int64_t x = 0; x < W; ++x) {
            int64_t best = gr[x];
            for (int64_t r = 1; r < W && r * r < best; ++r) {
                if (x - r >= 0 && gr[x - r] + r * r < best) best = gr[x - r] + r * r;
                if (x + r < W && gr[x + r] + r * r < best) best = gr[x + r] + r * r;
            }
            out[y * W + x] = sqrt((double)best);
        }
    }
    free(g);
    return 0;
}

/* silhouette.py:72-87 build_background: numpy reduces axis 0 of the
 * (K, H, W, C) float64 stack sequentially; population std, floor 2.0. */
OR_HOT void or_background(const uint8_t *frames, int64_t K, int64_t n, double *mean, double *std_) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double s = (double)frames[i];
        for (int64_t k = 1; k < K; ++k) s = s + (double)frames[k * n + i];
        const double m = s / (double)K;
        double v = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            const double d = (double)frames[k * n + i] - m;
            v = (k == 0) ? d * d : v + d * d;
        }
        const double sd = sqrt(v / (double)K);
        mean[i] = m;
        std_[i] = sd > 2.0 ? sd : 2.0; /* silhouette.py:86 np.maximum(std, STD_FLOOR) */
    }
}

/* silhouette.py:90-109 extract_silhouette. */
OR_HOT void or_extract(const uint8_t *frame, const double *mean, const double *std_,
                       const double *dm, int64_t npx, int64_t C, double theta_near,
                       double theta_far, double d_max, uint8_t *out) {
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < npx; ++p) {
        double dev = -INFINITY;
        for (int64_t c = 0; c < C; ++c) {
            const double x = (double)frame[p * C + c];
            const double d = fabs(x - mean[p * C + c]) / std_[p * C + c];
            if (d > dev || isnan(d)) dev = d;
        }
        double t = dm[p] / d_max;
        t = t < 1.0 ? t : 1.0; /* np.minimum(d / d_max, 1.0) */
        const double thr = theta_near + (theta_far - theta_near) * t;
        out[p] = dev > thr;
    }
}
