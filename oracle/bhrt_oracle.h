/*
 * bhrt_oracle.h — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference hot path (arXiv 2507.16165 `bhrt`,
 * /root/reference/proj) plus the north-star extensions (RK4 / RKF45
 * renderers, disk, spheres, checker sky, b-table). Every function cites the
 * reference file:line it follows.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) may load liboracle.so, and only as the checker or the
 * CPU baseline. The product path (paper_2507_16165_b200/) never calls it.
 *
 * Pinning: tests/test_oracle_*.py check this code against the reference's own
 * known-answer tests (proj/tests/test_geodesic.cpp, test_camera.cpp,
 * test_image.cpp, test_render.cpp, acceptance.cpp) and against golden vectors
 * produced by the compiled reference (oracle/_ref, tests/golden/).
 */
#ifndef BHRT_ORACLE_H
#define BHRT_ORACLE_H

#include "../include/bhrt_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* geodesic.cpp:31-33 / geodesic.hpp:79 */
void orc_ode_rhs(double phi, double u, double w, double mass, double out[2]);
/* camera.cpp:21-28 */
uint64_t orc_hash_counter(uint64_t seed, uint64_t a, uint64_t b, uint64_t c);
/* camera.cpp:30-43; returns 0 or BHRT_INVALID_ARGUMENT */
int orc_camera_basis(const bhrt_scene* s, double forward[3], double right[3], double up[3]);
/* camera.cpp:54-68 */
int orc_generate_ray(const bhrt_scene* s, int px, int py, int sample, double origin[3],
                     double dir[3]);
/* image.cpp:131-169 */
void orc_sample_direction(const uint8_t* rgb, int w, int h, const double dir[3], double out[3]);
/* geodesic.cpp:49-55; returns 1 when a basis exists, 0 when radial */
int orc_plane_basis(const double o[3], const double d[3], const double center[3], double e1[3],
                    double e2[3]);
/* geodesic.cpp:57-65; returns 0 or BHRT_INVALID_ARGUMENT (radial) */
int orc_initial_conditions(const double o[3], const double d[3], const double center[3],
                           double state[3]);
/* geodesic.cpp:67-69 */
double orc_step_dphi(double u, double epsilon);
/* geodesic.cpp:76-80 */
double orc_segment_dphi(double u, double w, double epsilon);
/* glibc 2.39 hypot (Borges' algorithm, non-FMA kernel) restated. */
double orc_hypot(double x, double y);
/* geodesic.cpp:84-162. Returns 0 ok, 1 StepSizeUnderflow (state in out),
 * BHRT_INVALID_ARGUMENT for dphi <= 0. `hint` may be NULL. steps/rejected
 * (may be NULL) are incremented. */
int orc_integrate_window(const double state[3], double dphi, double mass, double rel_tol,
                         double abs_tol, double* hint, double out[3], int* steps, int* rejected);
/* geodesic.cpp:164-238 on one ray. kind: 0 captured, 1 escaped, 2 stalled.
 * dir_out = escape direction. npoints = polyline length. last2 = the last two
 * polyline points (6 doubles). Returns 0, BHRT_INVALID_ARGUMENT or
 * BHRT_NUMERICAL. */
int orc_trace_reference(const double o[3], const double d[3], double mass, const double center[3],
                        double epsilon, double escape_radius, int max_windings, double rel_tol,
                        double abs_tol, int* kind, double dir_out[3], int* npoints, double last2[6],
                        int* steps, int* rejected);
/* geodesic.cpp:240-270 */
int orc_deflection_of_ray(const double o[3], const double d[3], double mass, const double center[3],
                          double epsilon, double escape_radius, int max_windings, double rel_tol,
                          double abs_tol, double* out);
/* geodesic.cpp:272-275 */
double orc_conserved_energy(double u, double w, double mass);
/* tests/oracles.hpp:23-30 */
void orc_rk4_step(double u, double w, double h, double mass, double out[2]);
/* tests/oracles.hpp:42-55: 0 captured, 1 escaped, 2 undecided */
int orc_classify(double u, double w, double mass, double escape_radius, double phi_budget,
                 double h);
/* One RKF45 step. Returns 1 if accepted. hnext gets
 * the controller's next step. */
int orc_rkf45_step(double u, double w, double h, double mass, double rel_tol, double abs_tol,
                   double max_step, double out[2], double* hnext);
/* RKF45 controller tables (host-computed, shared with the product by value). */
void orc_rkf45_factor_tables(double* grow, double* shrink, int* qmin, int* n);

/* One sample of one pixel: full scene semantics for every integrator.
 * rgb = the sample's linear colour. Returns 0, BHRT_NUMERICAL, or
 * BHRT_INVALID_ARGUMENT. */
int orc_trace_sample(const bhrt_scene* s, int px, int py, int sample, bhrt_ray_record* rec,
                     double rgb[3]);
/* render.cpp:22-49 */
int orc_shade_pixel(const bhrt_scene* s, int px, int py, uint8_t out[3], bhrt_ray_record* recs);
/* render.cpp:68-119 with a pthread dynamic row queue. */
int orc_render_rows(const bhrt_scene* s, int row_start, int row_end, int threads, uint8_t* out,
                    bhrt_ray_record* records, bhrt_status_info* info);
/* render.cpp:11-20 plus trace validation. */
int orc_validate_scene(const bhrt_scene* s, bhrt_status_info* info);
/* render.cpp:51-66 */
int orc_make_bands(int height, int workers, int* row_start, int* row_end, int capacity,
                   int* count);
/* Seeded sphere field, same definition as bhrt_make_spheres. */
int orc_make_spheres(uint64_t seed, int n, const double center[3], double shell_min,
                     double shell_max, double radius_min, double radius_max, bhrt_sphere* out);
void orc_scene_defaults(bhrt_scene* s);

/* Approximate mode (config 3): a table of INBOUND null
 * orbits u(psi) for b_e = table_b_max * e / (table_entries - 1), sampled at
 * psi_j = j * table_dpsi by RKF45 (scene tolerances), ending at capture
 * (u = 1/2M) or periapsis (u' = 0). Per entry: kind (0 captured, 1 escaping,
 * 2 undecided/truncated, 3 radial b = 0), n samples, ends = {psi_end, u_end,
 * w_end, psi_esc}, samples = (u, u') pairs. */
typedef struct orc_table orc_table;
orc_table* orc_table_build(const bhrt_scene* s);
void orc_table_free(orc_table* t);
int orc_table_entry(const orc_table* t, int e, int* kind, int* n, double ends[4], double* samples,
                    int cap);
/* Inbound psi where u = target on entry e (Hermite + Newton), -1 if unreachable. */
double orc_table_inbound_psi(const orc_table* t, int e, double target);

#ifdef __cplusplus
}
#endif

#endif
