// hbflow_gpu.hpp — C++ drop-in adapter: the reference's hot-path signatures,
// forwarded to the B200 library through the C ABI (include/hbgpu.h).
//
// This is the code a maintainer adds to the reference tree
// (/root/reference/proj) to move the HB-GLS hot path onto the GPU.  Every
// function has the exact signature of the reference function it replaces, so a
// call site switches by namespace only:
//   hbflow::assemble_residual      assembly.hpp:129-134
//   hbflow::assemble_tangent       assembly.hpp:138-141
//   hbflow::assemble_mass          assembly.hpp:145-146
//   TangentOperator::matvec        linalg.hpp:75           -> gpu::matvec(L, y, out)
//   hbflow::jacobi_preconditioner  linalg.hpp:84
//   hbflow::gmres_solve            linalg.hpp:111-115
//   hbflow::solve_harmonic         hb_solver.hpp:70-72
//   hbflow::solve_time             time_solver.hpp:51-54
// Device contexts are cached per Mesh (geometry, pattern, incidence lists
// are uploaded once); status codes are rethrown as the reference exceptions.
#pragma once

#include "hbflow/assembly.hpp"
#include "hbflow/hb_solver.hpp"
#include "hbflow/linalg.hpp"
#include "hbflow/time_solver.hpp"

#include <functional>
#include <span>
#include <vector>

namespace hbflow::gpu {

std::vector<double> assemble_residual(const Mesh& mesh, const std::vector<ElementGeometry>& geoms,
                                      const HarmonicState& state, const SpectralOperators& ops,
                                      const FluidProperties& props,
                                      const BoundaryConditionSet& bcs, const AssemblyConfig& cfg,
                                      int threads = 1);

void assemble_tangent(const Mesh& mesh, const std::vector<ElementGeometry>& geoms,
                      const HarmonicState& state, const FluidProperties& props,
                      const BoundaryConditionSet& bcs, const AssemblyConfig& cfg,
                      BlockSparseMatrix& P);

std::vector<double> assemble_mass(const Mesh& mesh, const std::vector<ElementGeometry>& geoms,
                                  double rho, const NodePattern& pattern);

/// TangentOperator::matvec on the device (uploads L.P / L.mass when they did
/// not come from gpu::assemble_tangent / gpu::assemble_mass).
void matvec(const TangentOperator& L, std::span<const double> y, std::span<double> out);

JacobiPreconditioner jacobi_preconditioner(const TangentOperator& L);

KrylovResult gmres_solve(const TangentOperator& L, std::span<const double> rhs,
                         const JacobiPreconditioner& pc, const KrylovConfig& cfg);

/// The generic overload (linalg.hpp:107-109): any host operator.  The Krylov
/// basis and its orthogonalisation live on the device; each application of
/// `apply` goes through host buffers.  A vector-only device context is cached
/// per vector length.
KrylovResult gmres_solve(const std::function<void(std::span<const double>, std::span<double>)>& apply,
                         std::span<const double> rhs, std::span<const double> inv_diag,
                         const KrylovConfig& cfg);

HbSolution solve_harmonic(const Mesh& mesh, const std::vector<ElementGeometry>& geoms,
                          const SpectralBasis& basis, const FluidProperties& props,
                          const BoundaryConditionSet& bcs, const SolverConfig& cfg);

/// Generalized-alpha time stepping (the paper's comparison baseline) on the
/// device: time_residual / time_tangent kernels, N = 1 L-matvec and GMRES.
TimeSolution solve_time(const CaseInputs& inputs, const TimeSolverConfig& cfg);

/// Drop the cached device context of a mesh.
void release(const Mesh& mesh);

}  // namespace hbflow::gpu
