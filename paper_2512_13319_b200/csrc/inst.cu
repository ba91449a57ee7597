// inst.cu -- one explicit instantiation of the solver per translation unit.
// Compiled once per (PM_R, PM_NX, PM_NY, PM_KIND, PM_K) by the build (see build.py):
//   PM_KIND 0 = LTI linear, 1 = time-varying linear, 2 = coordinated turn, 3 = Van der Pol,
//   4 = LTI linear with paper-faithful Euler blocks of PM_NSUB substeps.
#include "pmap_make.cuh"

namespace pmap_rt {
#if PM_KIND == 0
template Runner* make_lti<PM_R, PM_NX, PM_NY, PM_K, 0, ~0u, ~0u>(const double*, const double*, const double*,
                                                               const double*, const double*, const double*,
                                                               const double*, const double*, const double*,
                                                               const double*, const double*, const double*);
#if PM_NX == 4 && PM_NY == 2  // rank-2 diffusion (Wiener velocity): Woodbury node update, dense and masked
template Runner* make_lti<PM_R, PM_NX, PM_NY, PM_K, 2, ~0u, ~0u>(const double*, const double*, const double*,
                                                               const double*, const double*, const double*,
                                                               const double*, const double*, const double*,
                                                               const double*, const double*, const double*);
template Runner* make_lti<PM_R, PM_NX, PM_NY, PM_K, 2, pmap_rt::kWienerAMask, pmap_rt::kWienerUMask>(
    const double*, const double*, const double*, const double*, const double*, const double*, const double*,
    const double*, const double*, const double*, const double*, const double*);
template Runner* make_lti<PM_R, PM_NX, PM_NY, PM_K, 2, pmap_rt::kWienerAMask, pmap_rt::kWienerUMask,
                          pmap_rt::kWienerSMask>(const double*, const double*, const double*, const double*,
                                                 const double*, const double*, const double*, const double*,
                                                 const double*, const double*, const double*, const double*);
#endif
#elif PM_KIND == 1
template Runner* make_tv<PM_R, PM_NX, PM_NY, PM_K>(const PM_R*, const PM_R*, const PM_R*, const PM_R*, const PM_R*,
                                             const PM_R*, const PM_R*, const int64_t*, int, double, const double*,
                                             const double*);
#elif PM_KIND == 2
template Runner* make_nl<PM_R, 5, 2, 1, PM_K>(double, double, double, const double*, const double*, const double*,
                                              const double*);
#elif PM_KIND == 4  // Euler blocks (f2), n = PM_NSUB substeps, LTI
template Runner* make_euler<PM_R, PM_NX, PM_NY, PM_NSUB, PM_K>(const double*, const double*, const double*,
                                                             const double*, const double*, const double*,
                                                             const double*, const double*, const double*,
                                                             const double*);
#elif PM_KIND == 3
template Runner* make_nl<PM_R, 2, 1, 2, PM_K>(double, double, double, const double*, const double*, const double*,
                                              const double*);
#endif
}  // namespace pmap_rt
