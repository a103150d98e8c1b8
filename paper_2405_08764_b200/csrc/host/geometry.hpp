// Mesh / metric setup of the B200 framework (host side, as in the reference).
//
// Mirrors the reference's geometry interface (proj/include/patchdyn/geometry.hpp:
// 14-91) so a reference user finds the same types: a Mapping carries analytic
// forward map, inverse metrics and second derivatives; transform_coefficients
// produces the pointwise coefficients of the transformed equation (PAPER.md
// Eq. 8).  The arithmetic follows proj/src/geometry.cpp:93-125 in the same
// evaluation order so that the coefficient tables the device consumes are
// bit-identical to what the reference's PatchIntegrator samples
// (microsim.cpp:236-249).  Compiled with -ffp-contract=off.
#pragma once

#include <functional>
#include <stdexcept>
#include <string>

namespace pdb200 {

// Error types, same names and hierarchy as proj/include/patchdyn/errors.hpp:9-61;
// each carries the C-ABI status it maps to.
struct Error : std::runtime_error {
    int status;
    Error(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};
#define PDB200_ERROR(Name, code) \
    struct Name : Error {        \
        explicit Name(const std::string& m) : Error(code, m) {} \
    };
PDB200_ERROR(NonPositiveJacobian, 1)
PDB200_ERROR(DerivativeMismatch, 2)
PDB200_ERROR(MixedTermUnsupported, 3)
PDB200_ERROR(StabilityViolation, 4)
PDB200_ERROR(IndexOutOfRange, 6)
PDB200_ERROR(ShapeMismatch, 7)
PDB200_ERROR(InvalidStretch, 8)
PDB200_ERROR(MacroInstability, 12)
PDB200_ERROR(MacroPatchError, 13)
PDB200_ERROR(ValidationError, 15)
PDB200_ERROR(DeviceError, 100)
PDB200_ERROR(Unsupported, 101)
#undef PDB200_ERROR

namespace geometry {

enum class MapKind { Identity, Stretched, Polar, UserAnalytic };

struct PhysPoint {
    double x, y;
};
// derivatives of (x,y) with respect to (xi,eta)
struct InverseMetrics {
    double x_xi, x_eta, y_xi, y_eta;
};
struct SecondDerivs {
    double x_xixi, x_xieta, x_etaeta;
    double y_xixi, y_xieta, y_etaeta;
};

struct Mapping {
    MapKind kind = MapKind::Identity;
    double stretch = 0.0;
    std::function<PhysPoint(double, double)> forward;
    std::function<InverseMetrics(double, double)> metrics;
    std::function<SecondDerivs(double, double)> second;
};

Mapping identity_map();
Mapping stretched_map(double lambda);  // x = xi + lambda/pi sin(pi xi), same in eta
Mapping polar_map();                   // (xi,eta) = (theta,r), (x,y) = (r sin, r cos): J = +r
Mapping user_analytic_map(std::function<PhysPoint(double, double)> fwd,
                          std::function<InverseMetrics(double, double)> met,
                          std::function<SecondDerivs(double, double)> sec);

// l u_t + alpha u_xx + beta u_yy + gamma u_x + nu u_y + omega u = phi
struct PhysicalCoefficients {
    using Fn = std::function<double(double, double, double)>;
    Fn alpha, beta, gamma, nu, omega, phi;
    double l = 1.0;
};
PhysicalCoefficients cdr_coefficients(PhysicalCoefficients::Fn Dx, PhysicalCoefficients::Fn Dy,
                                      PhysicalCoefficients::Fn vx, PhysicalCoefficients::Fn vy,
                                      PhysicalCoefficients::Fn source);

// l u_t + a u_xixi + b u_xieta + c u_etaeta + d u_xi + e u_eta + f u = g
struct TransformedCoefficients {
    double a, b, c, d, e, f, g;
    double R, S;
};

double jacobian(const Mapping& m, double xi, double eta);
TransformedCoefficients transform_coefficients(const Mapping& m, const PhysicalCoefficients& p,
                                               double xi, double eta, double t);

} // namespace geometry
} // namespace pdb200
